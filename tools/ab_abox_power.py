"""Power-aware A/B at the cfg4 shape: 128-B (a_box 1) vs 256-B (a_box 2) row visits of A. Long runs
(2 s per variant per round, 1 s rest), interleaved rounds; ms per call and effective SM clock."""
import json
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

m, k, n = 1 << 22, 4096, 256
A = shg.synth('gauss', 2, 0x100, m, k)
Om = shg.gen_omega(k, n)
Y = torch.empty((m, n), device='cuda')
V = [('abox1', {'a_box': 1}), ('abox2', {'a_box': 2})]
prof = torch.zeros((148, 16), dtype=torch.int64, device='cuda')
for rnd in range(3):
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
        t = dict(tune)
        t['prof'] = prof.data_ptr()
        shg.shgemm(A, Om, out=Y, tune=t)
        torch.cuda.synchronize()
        cyc = float(prof[:, 0].max())
        print(json.dumps({"round": rnd, "variant": name, "ms": ms, "tflops": 2.0 * m * n * k / ms / 1e9,
                          "cycles_per_call": cyc}), flush=True)
