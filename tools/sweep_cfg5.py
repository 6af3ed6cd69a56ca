"""BASELINE config 5: the n sweep at m = k = 32768 across the HBM -> tensor-core ridge. Per n: median
of 3 rounds of back-to-back calls (gen_omega + shgemm, the hot path), TFLOP/s, GB/s and the fraction
of min(tensor/2, AI x HBM) with the burst and the sustained tensor peak (MEASURED_PEAKS.json)."""
import json
import statistics
import sys

import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
import paper_2304_04612_b200 as shg  # noqa: E402

hbm, tc_burst, tc_sus, _ = bench.load_peaks()
m = k = 32768
A = shg.synth("gauss", 2, 0x101, m, k)
for n in (16, 32, 64, 128, 192, 256, 272, 384, 512, 1024, 2048, 4096):
    Om = shg.gen_omega(k, n)
    Y = torch.empty((m, n), device="cuda")
    reps = max(3, int(200 / (0.001 * n + 0.7)))  # ~0.2 s per round
    for _ in range(3):
        shg.gen_omega(k, n, seed=0)
        shg.shgemm(A, Om, out=Y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            shg.gen_omega(k, n, seed=0)
            shg.shgemm(A, Om, out=Y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    ms = statistics.median(ts)
    fl, by = 2.0 * m * k * n, 4.0 * m * k + 2.0 * k * n + 4.0 * m * n
    tf = fl / ms / 1e9
    ai_bw = fl / by * hbm / 1e3
    print(json.dumps({"n": n, "ms": ms, "tflops": tf, "gbs": by / ms / 1e6, "plan_bn": shg.plan(m, n, k)["bn"],
                      "bound": "tensor" if tc_burst / 2 < ai_bw else "hbm",
                      "frac_burst": tf / min(tc_burst / 2, ai_bw), "frac_sustained": tf / min(tc_sus / 2, ai_bw)}),
          flush=True)
    del Om, Y
    torch.cuda.empty_cache()
