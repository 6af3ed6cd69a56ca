"""Round-2 fuzz of the RandNLA harness against the oracle pipelines (north_star: residuals within
1e-4 relative of the FP32 oracle pipeline, reading R10): random-shape RSVD (prescribed spectra,
both GEMM/factor variants) and RP-HOSVD (noisy Alg-3 tensors, odd dims, both variants).
Usage: python tools/fuzz_pipelines.py LO HI."""
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, '.')
import oracle  # noqa: E402,F401
from oracle import pipelines as opl  # noqa: E402
import synth  # noqa: E402
from paper_2304_04612_b200 import pipelines as pl  # noqa: E402


def run(i):
    r = np.random.default_rng(800000 + i)
    if i % 2 == 0:
        N = int(r.integers(64, 1500))
        p = int(r.integers(2, min(64, N // 4)))
        s = int(r.integers(2, 20))
        kind = ["exp", "linear"][int(r.integers(0, 2))]
        A = synth.spectrum_matrix(synth.spectrum(kind, N, p, 10.0 ** -r.uniform(1, 3)), seed=i)
        variant = [{}, {"gemm": "tcec", "factor": "gram"}, {"gemm": "tcec"}][int(r.integers(0, 3))]
        res = pl.rsvd(torch.from_numpy(A).cuda(), p, s, seed=i, **variant)
        e_gpu = pl.reconstruction_error(torch.from_numpy(A).cuda(), res["U"], res["S"], res["V"])
        e_or = opl.rsvd(A, p, s, seed=i, precision="f32")["residual"]
    else:
        dims = tuple(int(x) for x in r.integers(6, 70, size=int(r.integers(3, 5))))
        ranks = tuple(int(min(d, r.integers(3, 12))) for d in dims)
        pad = int(r.integers(1, 3))
        T = synth.alg3_tensor(dims, ranks, pad=pad, seed=i, noise=1e-2)
        variant = [{}, {"gemm": "tcec", "factor": "gram"}][int(r.integers(0, 2))]
        res = pl.rp_hosvd(torch.from_numpy(T).cuda(), ranks, seed=i, **variant)
        e_gpu = pl.hosvd_error(torch.from_numpy(T).cuda(), res["core"], res["Q"])
        e_or = opl.rp_hosvd(T, ranks, seed=i, precision="f32")["residual"]
    assert e_or > 1e-6, e_or
    assert abs(e_gpu - e_or) <= 1e-4 * e_or, (e_gpu, e_or)


lo, hi = int(sys.argv[1]), int(sys.argv[2])
fails = 0
for i in range(lo, hi):
    try:
        run(i)
    except Exception as e:
        fails += 1
        print("FAIL", i, repr(e)[:300], flush=True)
        traceback.print_exc(limit=3)
print(f"fuzz_pipelines done: {hi - lo} cases, {fails} failures", flush=True)
