"""Re-run fuzz cases of tests/test_gpu_fuzz.py and print the worst elements against the oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle as orc  # noqa: E402
orc.build()
import paper_2304_04612_b200 as shg  # noqa: E402
import test_gpu_fuzz as tf  # noqa: E402
from gpu_common import omega_bits, to_np, U32  # noqa: E402

for i in map(int, sys.argv[1:]):
    m, k, n, kind, mmajor, tune, dist, tiled, scale = tf.case(i)
    print("case", i, (m, k, n, kind, mmajor, tune, dist, tiled, scale))
    r = np.random.default_rng(i)
    A = (r.standard_normal((m, k)) * scale).astype(np.float32)
    Om = shg.gen_omega(k, n, seed=i, dist=dist)
    print("plan", shg.plan(m, n, k, tune or None))
    for variant in ("asis", "kmajor", "simt"):
        if variant == "asis" and mmajor:
            mp = (m + 3) // 4 * 4
            buf = torch.zeros((k, mp), dtype=torch.float32, device="cuda")
            buf[:, :m] = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
            Y = shg.shgemm_at(buf[:, :m], Om, tune=tune or None)
        elif variant == "simt":
            Y = shg.shgemm(torch.from_numpy(A).cuda(), Om, tune={"force_simt": 1})
        else:
            Y = shg.shgemm(torch.from_numpy(A).cuda(), Om, tune=tune or None)
        torch.cuda.synchronize()
        ob = omega_bits(Om)
        Yn = to_np(Y).astype(np.float64)
        y64 = orc.gemm_y64(A, ob)
        W = np.abs(orc.f16_bits_as_float(ob).astype(np.float64))
        bound = 1.2 * (k / 8 + 3) * U32 * (np.abs(A).astype(np.float64) @ W)
        ratio = np.abs(Yn - y64) / np.maximum(bound, 1e-300)
        idx = np.unravel_index(np.argmax(ratio), ratio.shape)
        bad = np.argwhere(ratio > 1)
        print(variant, "worst", float(ratio.max()), "at", idx, "gpu", Yn[idx], "y64", y64[idx], "bound", bound[idx],
              "n_bad", len(bad), "rows", np.unique(bad[:, 0])[:10] if len(bad) else None,
              "cols", np.unique(bad[:, 1])[:20] if len(bad) else None)
        if len(bad):
            ii, jj = idx
            print("   A row", A[ii], "\n   Om col", orc.f16_bits_as_float(ob[:, jj]))
