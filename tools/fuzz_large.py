"""Randomised sweep at larger shapes than tests/test_gpu_fuzz.py (m up to 40000, k up to 20000,
n up to 1100, so several N tiles, CTA pairs, wide tiles, split-K and the tensor-core path on every
kind): Y on 24 sampled rows (first/last + random) against the oracle bars (tests/gpu_common.py,
DESIGN §3, R20, R22). Usage: python tools/fuzz_large.py LO HI."""
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle as orc  # noqa: E402
orc.build()
import paper_2304_04612_b200 as shg  # noqa: E402
from gpu_common import U32, check_bars, omega_bits, to_np  # noqa: E402


def case(i):
    r = np.random.default_rng(90000 + i)
    m = int(r.integers(1, 40000))
    k = int(r.integers(1, 20000))
    n = int(r.choice([int(r.integers(1, 1100)), 256, 272, 288, 512, 544, 1024]))
    kind = ["fp16", "fp16", "tf32", "tcec"][i % 4]
    mmajor = bool(r.integers(0, 2))
    tune = {}
    if r.random() < 0.25:
        tune["split_k"] = int(r.integers(1, 5))
    if r.random() < 0.2:
        tune["pair"] = int(r.integers(1, 3))
    if r.random() < 0.25:
        tune["stream_k"] = int(r.integers(1, 3))     # forced stream-K / whole tiles (0 = auto)
    if r.random() < 0.2:
        tune["a_mcast"] = int(r.choice([1, 2, 4]))   # A multicast forced off / 2 / 4 pairs (0 = auto)
    row_omega = r.random() < 0.3                      # SURVEY §8(b)'s row-major Omega
    dist = int(r.integers(0, 4)) if kind != "tcec" else 0
    scale = float(np.exp(r.uniform(-3, 3)))
    return m, k, n, kind, mmajor, tune, dist, scale, row_omega


def run(i):
    m, k, n, kind, mmajor, tune, dist, scale, row_omega = case(i)
    g = torch.Generator(device="cuda").manual_seed(i)
    A = torch.randn(m, k, device="cuda", generator=g) * scale
    if mmajor:
        mp = (m + 3) // 4 * 4
        buf = torch.zeros((k, mp), device="cuda")
        buf[:, :m] = A.t()
        Ad = buf[:, :m].t()
    else:
        Ad = A
    rr = np.random.default_rng(i)
    rows = np.unique(np.concatenate([[0, m - 1], rr.integers(0, m, 22)]))
    ridx = torch.from_numpy(rows).cuda()
    try:
        if kind == "tcec":
            B = torch.randn(k, n, device="cuda", generator=g)
            C = shg.tcec_sgemm(Ad, B, tune=tune or None)
            torch.cuda.synchronize()
            An, Bn, Cn = to_np(A[ridx]), to_np(B), to_np(C[ridx]).astype(np.float64)
            y64 = orc.gemm_y64_f32b(An, Bn)
            Aa, Ba = np.abs(An).astype(np.float64), np.abs(Bn).astype(np.float64)
            bound = 1.2 * ((k / 8 + 9) * U32 * (Aa @ Ba) + 2.0 ** -35 * ((Aa < 2.0 ** -13) @ Ba + Aa @ (Ba < 2.0 ** -13)))
            assert np.all(np.abs(Cn - y64) <= bound), float(np.max(np.abs(Cn - y64) / np.maximum(bound, 1e-300)))
            assert orc.relative_error(Cn, y64) <= 1e-5
            return
        Om = shg.gen_omega(k, n, seed=i, dist=dist, layout="row" if row_omega else "col")
        if mmajor:
            Y = shg.shgemm_at(Ad.t(), Om, tune=tune or None, tc=kind)
        else:
            Y = shg.shgemm(Ad, Om, tune=tune or None, tc=kind)
        torch.cuda.synchronize()
        if kind == "fp16" and not mmajor and shg.plan(m, n, k, tune or None)["a_mcast"] > 1:
            # A multicast (auto or forced): bitwise equal to per-pair loads on the same whole tiles
            Y0 = shg.shgemm(Ad, Om, tune=dict(tune, a_mcast=1, split_k=1))
            torch.cuda.synchronize()
            assert torch.equal(Y.view(torch.int32), Y0.view(torch.int32)), "a_mcast not bitwise"
    except shg.SHGError as err:
        assert "INVALID" in str(err) and tune, err
        return
    ob = omega_bits(Om)
    An = to_np(A[ridx])
    if not np.any(orc.gemm_y64(An, ob)):
        return
    check_bars(orc, An, ob, to_np(Y[ridx]), ratio=2.0 if k >= 16 else float("inf"))


lo, hi = int(sys.argv[1]), int(sys.argv[2])
fails = 0
for i in range(lo, hi):
    try:
        run(i)
    except Exception as e:
        fails += 1
        print("FAIL", i, case(i), repr(e)[:300], flush=True)
    torch.cuda.empty_cache()
print(f"fuzz_large done: {hi - lo} cases, {fails} failures", flush=True)
