"""Wave quantisation vs split-K on the cfg5 shapes: per-call device time (back to back, median of
20) for split_k 1..4 at m = k = 32768 and n = 64..256, and cfg2's 16384^2 x 272."""
import json
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

ws = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def med(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


for m, k, n in [(32768, 32768, 64), (32768, 32768, 128), (32768, 32768, 192), (32768, 32768, 256),
                (16384, 16384, 272), (65536, 32768, 128)]:
    A = shg.synth("gauss", 2, 0x100, m, k)
    Om = shg.gen_omega(k, n)
    Y = torch.empty(m, n, device="cuda")
    r = {"m": m, "k": k, "n": n, "auto": shg.plan(m, n, k)}
    for sk in (1, 2, 3, 4):
        t = {"split_k": sk}
        try:
            ms = med(lambda: shg.shgemm(A, Om, out=Y, tune=t, workspace=ws))
        except shg.SHGError as e:
            ms = None
        r[f"sk{sk}_ms"] = ms
        if ms:
            r[f"sk{sk}_tflops"] = 2 * m * n * k / ms / 1e9
    print(json.dumps(r), flush=True)
    del A
