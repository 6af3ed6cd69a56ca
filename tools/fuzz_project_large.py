"""Randomised project() sweep on larger C-order tensors (3-4 modes, up to ~1.5e8 elements, every
unfolding view, separate or in-kernel Omega, FP16 / TF32): W on 12 sampled rows against the oracle
(the oracle's own Omega_(mode), stream_id = mode). Usage: python tools/fuzz_project_large.py LO HI."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle as orc  # noqa: E402
orc.build()
import paper_2304_04612_b200 as shg  # noqa: E402
from gpu_common import check_bars, to_np  # noqa: E402


def case(i):
    r = np.random.default_rng(70000 + i)
    nd = int(r.integers(3, 5))
    while True:
        dims = tuple(int(x) for x in np.exp(r.uniform(np.log(2), np.log(1500), nd)).astype(int))
        tot = int(np.prod(dims))
        if 1e5 <= tot <= 1.5e8:
            break
    mode = int(r.integers(0, nd))
    n = int(r.choice([8, 16, 24, 33, 64, 100, 128]))
    K = tot // dims[mode]
    while K * n > 6e7 and n > 8:
        n //= 2
    dist = int(r.integers(0, 4))
    tc = "tf32" if r.random() < 0.25 else "fp16"
    inkernel = bool(r.integers(0, 2)) and tc == "fp16"
    return dims, mode, n, dist, tc, inkernel


def run(i):
    dims, mode, n, dist, tc, inkernel = case(i)
    K = int(np.prod(dims)) // dims[mode]
    if K * n > 6e7:
        return
    g = torch.Generator(device="cuda").manual_seed(i)
    T = torch.randn(*dims, device="cuda", generator=g)
    shg.set_inkernel_omega(inkernel)
    try:
        W = shg.project(T, mode, n, seed=i, dist=dist, tc=tc)
        torch.cuda.synchronize()
    finally:
        shg.set_inkernel_omega(False)
    I = dims[mode]
    rows = np.unique(np.concatenate([[0, I - 1], np.random.default_rng(i).integers(0, I, 10)]))
    ridx = torch.from_numpy(rows).cuda()
    U = to_np(torch.movedim(T, mode, 0)[ridx].reshape(len(rows), -1))
    ob = orc.omega_f16(K, n, seed=i, dist=dist, stream_id=mode)
    if not np.any(orc.gemm_y64(U, ob)):
        return
    check_bars(orc, U, ob, to_np(W[ridx]), ratio=2.0 if K >= 16 else float("inf"))


lo, hi = int(sys.argv[1]), int(sys.argv[2])
fails = 0
for i in range(lo, hi):
    try:
        run(i)
    except Exception as e:
        fails += 1
        print("FAIL", i, case(i), repr(e)[:300], flush=True)
    torch.cuda.empty_cache()
print(f"fuzz_project_large done: {hi - lo} cases, {fails} failures", flush=True)
