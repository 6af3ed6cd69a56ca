"""Sustained tensor throughput under the power cap: the same MMA work as 1 x N=256 or 2 x N=128
per K step (shg_probe_mma_energy); each case ~2 s after a 1 s rest, cases interleaved."""
import ctypes
import json
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

L = shg.lib()
L.shg_probe_mma_energy.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                   ctypes.c_void_p]
L.shg_probe_mma_energy.restype = ctypes.c_int
clusters = 74
out = torch.zeros(clusters, dtype=torch.int64, device='cuda')
cases = [(256, 1), (256, 2), (128, 1)]
for rnd in range(2):
    for n, parts in cases:
        iters = 400000 * 256 // n
        time.sleep(1.0)
        for _ in range(1):
            assert L.shg_probe_mma_energy(n, parts, iters // 10, shg._p(out), clusters, shg._stream()) == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert L.shg_probe_mma_energy(n, parts, iters, shg._p(out), clusters, shg._stream()) == 0
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        flops = 2.0 * 256 * n * 16 * iters * clusters
        cyc = float(out.max())
        print(json.dumps({"round": rnd, "n": n, "parts": parts, "ms": ms, "tflops": flops / ms / 1e9,
                          "cycles_per_kstep": cyc / iters, "ghz_eff": cyc / ms / 1e6}), flush=True)
