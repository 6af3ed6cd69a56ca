"""Randomised (fixed-seed, reproducible) sweep of shapes x layouts x kinds x tunables through the C ABI
against the oracle bars of DESIGN.md §3: 240 cases, each a different combination of m, k, n (ragged
in every dimension), SHGEMM-FP16 / -TF32 / TCEC-SGEMM, K-major / M-major A, single CTAs / pairs,
split-K, wide tiles, k-tiled Omega and the Omega distributions."""
import numpy as np
import pytest

from gpu_common import U32, check_bars, omega_bits, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def shg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_04612_b200 import _build
    _build.build()
    import paper_2304_04612_b200 as m
    return m


def case(i):
    r = np.random.default_rng(1000 + i)
    m = int(r.integers(1, 1500))
    k = int(r.integers(1, 3000))
    n = int(r.choice([int(r.integers(1, 300)), 16, 32, 64, 128, 256, 272, 288]))
    kind = ["fp16", "fp16", "tf32", "tcec"][i % 4]
    mmajor = bool(r.integers(0, 2))
    tune = {}
    if r.random() < 0.3:
        tune["split_k"] = int(r.integers(1, 6))
    if r.random() < 0.2:
        tune["pair"] = int(r.integers(1, 3))
    if r.random() < 0.25:
        tune["stream_k"] = int(r.integers(1, 3))     # forced stream-K / whole tiles (0 = auto)
    row_omega = r.random() < 0.3                      # SURVEY §8(b)'s row-major Omega
    dist = int(r.integers(0, 4)) if kind != "tcec" else 0
    tiled = kind == "fp16" and not mmajor and k % 4 == 0 and r.random() < 0.3
    scale = float(np.exp(r.uniform(-4, 4)))
    return m, k, n, kind, mmajor, tune, dist, tiled, scale, row_omega


@pytest.mark.parametrize("i", range(240))
def test_fuzz(shg, orc, i):
    m, k, n, kind, mmajor, tune, dist, tiled, scale, row_omega = case(i)
    r = np.random.default_rng(i)
    A = (r.standard_normal((m, k)) * scale).astype(np.float32)
    # the M-major path needs a 16-B aligned row pitch for the tensor-core route; pad the stored
    # transpose so it takes it (ragged m otherwise exercises the CUDA-core fallback, also fine)
    def dev_A():
        if not mmajor:
            return torch.from_numpy(A).cuda()
        mp = (m + 3) // 4 * 4
        buf = torch.zeros((k, mp), dtype=torch.float32, device="cuda")
        buf[:, :m] = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
        return buf[:, :m].t()             # (m, k) view with stride (1, mp): MN-major
    try:
        if kind == "tcec":
            B = (r.standard_normal((k, n)) * np.exp(r.uniform(-3, 3))).astype(np.float32)
            C = to_np(shg.tcec_sgemm(dev_A(), torch.from_numpy(B).cuda(), tune=tune or None))
            y64, y32 = orc.gemm_y64_f32b(A, B), orc.gemm_y32_f32b(A, B)
            e, e32 = orc.relative_error(C, y64), orc.relative_error(y32, y64)
            # DESIGN R20: TCEC's elementwise bar is SHGEMM's + 6u (B's split, Eq 9's dropped term)
            Aa, Ba = np.abs(A).astype(np.float64), np.abs(B).astype(np.float64)
            bound = 1.2 * ((k / 8.0 + 9.0) * U32 * (Aa @ Ba) +
                           2.0 ** -35 * ((Aa < 2.0 ** -13) @ Ba + Aa @ (Ba < 2.0 ** -13)))
            assert np.all(np.abs(C - y64) <= bound + 1e-300)
            assert e <= 1e-5 and (k < 16 or e <= 2 * e32), (e, e32)
            return
        Om = shg.gen_omega(k, n, seed=i, dist=dist, layout="row" if row_omega else "col")
        Ad = dev_A()
        if tiled:
            Y = shg.shgemm_tiled(Ad, shg.gen_omega_tiled(k, n, seed=i, dist=dist), n, tune=tune or None)
        elif mmajor:
            Y = shg.shgemm_at(Ad.t(), Om, tune=tune or None, tc=kind)
        else:
            Y = shg.shgemm(Ad, Om, tune=tune or None, tc=kind)
        torch.cuda.synchronize()
    except shg.SHGError as err:       # only invalid tunables for the shape may be rejected
        assert "INVALID" in str(err) and tune, err
        return
    ob = omega_bits(Om)
    if float(np.abs(orc.f16_bits_as_float(ob)).max()) == 0.0 or min(m, n) == 0:
        return
    # exact-zero rows/cols (sparse Omega with k small) make the relative bars degenerate
    y64 = orc.gemm_y64(A, ob)
    if not np.any(y64):
        return
    # the ratio-to-naive-FP32 bar only for k >= 16: below that the split's 1-ulp representation loss
    # (25% of elements) dominates a naive error that is itself near zero; the
    # elementwise (k/8 + 3) u |A||Omega| bar and the 1e-5 bar still apply
    check_bars(orc, A, ob, to_np(Y), ratio=2.0 if k >= 16 else float("inf"))


@pytest.mark.parametrize("i", range(48))
def test_fuzz_project(shg, orc, i):
    """Random C-order tensors (2-4 modes, ragged extents) through project(): every unfolding view
    (mode 0, 3-D K-major, copied middle modes, M-major last mode), k-tiled Omega, the separate or the
    in-kernel generator, every distribution; W against the oracle bars on the unfolding."""
    from oracle import pipelines as opl
    r = np.random.default_rng(5000 + i)
    nd = int(r.integers(2, 5))
    dims = tuple(int(x) for x in r.integers(2, 40, size=nd))
    while int(np.prod(dims)) < 2000:
        dims = tuple(d * 2 for d in dims)
    mode = int(r.integers(0, nd))
    n = int(r.choice([8, 16, 33, 64, 100]))
    dist = int(r.integers(0, 4))
    inkernel = bool(r.integers(0, 2))
    T = r.standard_normal(dims).astype(np.float32)
    prev = shg.get_inkernel_omega()
    shg.set_inkernel_omega(inkernel)
    try:
        W = to_np(shg.project(torch.from_numpy(T).cuda(), mode, n, seed=i, dist=dist))
    finally:
        shg.set_inkernel_omega(prev)
    Ai = np.ascontiguousarray(opl.unfold(T, mode))
    K = Ai.shape[1]
    ob = orc.omega_f16(K, n, seed=i, dist=dist, stream_id=mode)
    if not np.any(orc.gemm_y64(Ai, ob)):
        return
    check_bars(orc, Ai, ob, W, ratio=2.0 if K >= 16 else float("inf"))
