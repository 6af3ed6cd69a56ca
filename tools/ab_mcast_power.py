"""Power-aware A/B at the cfg4 shape: Omega multicast 1 / 2 / 3 pairs per cluster. 100-call runs
(~2 s) per variant per round after a 1 s rest, 5 interleaved rounds; ms per call and SM clock."""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

m, k, n = 1 << 22, 4096, 256
A = shg.synth('gauss', 2, 0x100, m, k)
Om = shg.gen_omega(k, n)
Y = torch.empty((m, n), device='cuda')
V = [('mc1', {'omega_mcast': 1}), ('mc2', {'omega_mcast': 2}), ('mc3', {'omega_mcast': 3})]
prof = torch.zeros((148, 16), dtype=torch.int64, device='cuda')
res = {name: [] for name, _ in V}
for rnd in range(5):
    for name, tune in V:
        time.sleep(1.0)
        for _ in range(3):
            shg.shgemm(A, Om, out=Y, tune=tune)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 100
        s.record()
        for _ in range(reps):
            shg.shgemm(A, Om, out=Y, tune=tune)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        res[name].append(ms)
        print(json.dumps({"round": rnd, "variant": name, "ms": ms, "tflops": 2.0 * m * n * k / ms / 1e9}), flush=True)
print(json.dumps({name: statistics.median(v) for name, v in res.items()}))
