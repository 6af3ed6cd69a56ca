"""GPU parity tests for SHGEMM-TF32 (Eqs 14-17 with toLow = TF32, Omega FP16 in
memory, widened exactly to TF32 for the tensor cores), through the C ABI, against the oracle:
the device split bit-exact on all 2^32 FP32 patterns, identity-Omega and exact-integer cases
bit-exact, and the north_star bars elsewhere, including A far outside the FP16 range (A_Cauchy,
P:699-706) where SHGEMM-FP16 fails by design."""
import numpy as np
import pytest

import synth
from gpu_common import check_bars, omega_bits, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def shg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_04612_b200 import _build
    _build.build()
    import paper_2304_04612_b200 as m
    assert m.device_supported(), "device is not sm_100"
    return m


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run(shg, A, k, n, seed=0, dist=0, tune=None):
    Om = shg.gen_omega(k, n, seed=seed, dist=dist)
    Y = shg.shgemm(cuda(A), Om, tune=tune, tc="tf32")
    torch.cuda.synchronize()
    return omega_bits(Om), to_np(Y)


def test_split_tf32_exhaustive_all_fp32(shg, orc):
    """Device TF32 split (the mainloop's device function) == oracle on all 2^32 FP32 patterns
    (NaN inputs: NaN class)."""
    chunk = 1 << 28
    for c in range((1 << 32) // chunk):
        lo_pat = c * chunk
        bits = torch.arange(lo_pat, lo_pat + chunk, dtype=torch.int64, device="cuda").to(torch.int32)
        hi, lo = shg.split_tf32(bits.view(torch.float32))
        hi_np = to_np(hi).view(np.uint32)
        lo_np = to_np(lo).view(np.uint32)
        a_np = np.arange(lo_pat, lo_pat + chunk, dtype=np.uint64).astype(np.uint32).view(np.float32)
        rhi, rlo = orc.split_tf32(a_np)

        def isnan(u):
            return (u & 0x7FFFFFFF) > 0x7F800000
        ok_hi = (hi_np == rhi) | (isnan(hi_np) & isnan(rhi))
        ok_lo = (lo_np == rlo) | (isnan(lo_np) & isnan(rlo))
        assert ok_hi.all(), hex(int(a_np.view(np.uint32)[~ok_hi][0]))
        assert ok_lo.all(), hex(int(a_np.view(np.uint32)[~ok_lo][0]))


@pytest.mark.parametrize("scale", [7.0, 1e30, 1e-30])
def test_identity_omega_reconstructs_tf32_split(shg, orc, scale):
    """Omega = [I; 0]: Y[i][j] = RN_f32(hi + lo 2^-11) of A[i][j] exactly, at any FP32 magnitude —
    checks the tf32 MMA, the scale-input-d fold of lo and the promotion end to end."""
    m, k, n = 256, 192, 128
    A = (synth.gaussian(m, k, seed=3).astype(np.float64) * scale).astype(np.float32)
    eye = np.eye(k, n, dtype=np.float32).astype(np.float16)
    Om = torch.from_numpy(np.ascontiguousarray(eye.T)).cuda().t()
    Y = to_np(shg.shgemm(cuda(A), Om, tc="tf32"))
    hi, lo = orc.split_tf32(A[:, :n])
    rec = hi.view(np.float32).astype(np.float64) + lo.view(np.float32).astype(np.float64) * 2.0 ** -11
    rec = rec.reshape(m, n).astype(np.float32)
    assert np.array_equal(Y, rec)
    frac = np.mean(Y != A[:, :n])
    assert 0.15 < frac < 0.35


def test_exact_integer_case_bitwise(shg, orc):
    m, k, n = 300, 2048, 64
    A = synth.small_int_matrix(m, k, seed=5)
    om, Y = _run(shg, A, k, n, seed=3, dist=1)
    assert np.array_equal(Y.astype(np.float64), orc.gemm_y64(A, om))


CASES = [
    (512, 512, 32, "spectrum"),    # BASELINE config 1
    (512, 512, 32, "normal"),
    (300, 1000, 50, "uniform"),
    (129, 65, 17, "normal"),
    (1000, 777, 272, "normal"),
    (640, 4096, 256, "normal"),
    (384, 16384, 64, "normal"),    # split-K
]


@pytest.mark.parametrize("m,k,n,kind", CASES)
def test_shgemm_tf32_bars(shg, orc, m, k, n, kind):
    if kind == "spectrum":
        A = synth.spectrum_matrix(synth.spectrum("exp", m, 22, 1e-2), seed=1)[:, :k]
    elif kind == "normal":
        A = synth.gaussian(m, k, seed=m + k)
    else:
        A = synth.uniform(m, k, seed=m + k)
    om, Y = _run(shg, A, k, n)
    check_bars(orc, A, om, Y)


@pytest.mark.parametrize("tune", [{"force_simt": 1}, {"split_k": 3}, {"bn": 64}, {"pair": 1}, {"pair": 2},
                                  {"pair": 1, "bn": 144}, {"a_box": 2}, {"max_ctas": 5}])
def test_shgemm_tf32_tunables(shg, orc, tune):
    m, k, n = 400, 1504, 200          # k % 64 == 32: a half-stage tail (and k % 32 == 0 for a_box 2)
    A = synth.gaussian(m, k, seed=2)
    om, Y = _run(shg, A, k, n, tune=tune)
    check_bars(orc, A, om, Y)


def test_full_exponent_range_cauchy(shg, orc):
    """A_Cauchy-like input (|a| > 65504): SHGEMM-FP16 flags non-finite rows,
    SHGEMM-TF32 stays finite and inside the bars (the point of the TF32 variant)."""
    A = synth.cauchy_like(256, seed=0)
    assert np.abs(A).max() > 65504
    Om = shg.gen_omega(256, 32, seed=0)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    shg.shgemm(cuda(A), Om, nonfinite=flag)
    assert int(flag.item()) == 1
    flag.zero_()
    Y = to_np(shg.shgemm(cuda(A), Om, nonfinite=flag, tc="tf32"))
    assert int(flag.item()) == 0
    check_bars(orc, A, omega_bits(Om), Y)


def test_wide_dynamic_range_rows(shg, orc):
    """Rows scaled from 2^-100 to 2^100: relative accuracy per row is scale-free in TF32."""
    m, k, n = 256, 1024, 64
    A = synth.gaussian(m, k, seed=11).astype(np.float64)
    A *= np.exp2(np.linspace(-100, 100, m))[:, None]
    A = A.astype(np.float32)
    om, Y = _run(shg, A, k, n)
    y64 = orc.gemm_y64(A, om)
    W = np.abs(orc.f16_bits_as_float(om).astype(np.float64))
    bound = 1.2 * (k / 8.0 + 3.0) * 2.0 ** -24 * (np.abs(A).astype(np.float64) @ W)
    assert np.all(np.abs(Y - y64) <= bound)


def test_tf32_mmajor_and_project(shg, orc):
    """M-major A (shgemm_at) and all project() modes with tc='tf32'."""
    from oracle import pipelines as pl
    m, k, n = 700, 1024, 144
    A = synth.gaussian(m, k, seed=21)
    Om = shg.gen_omega(k, n, seed=4)
    Y = to_np(shg.shgemm_at(torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), Om, tc="tf32"))
    check_bars(orc, A, omega_bits(Om), Y)
    dims = (96, 128, 256)
    T = synth.gaussian(int(np.prod(dims)), 1, seed=12).reshape(dims)
    Tt = cuda(T)
    for mode in range(3):
        W = to_np(shg.project(Tt, mode, 48, seed=9, tc="tf32"))
        U = np.ascontiguousarray(pl.unfold(T, mode))
        check_bars(orc, U, orc.omega_f16(U.shape[1], 48, seed=9, stream_id=mode), W)


def test_tf32_deterministic_and_plan(shg):
    A = cuda(synth.gaussian(700, 3000, seed=4))
    Om = shg.gen_omega(3000, 200, seed=1)
    Y1 = shg.shgemm(A, Om, tc="tf32").clone()
    Y2 = shg.shgemm(A, Om, tc="tf32")
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    p = shg.plan(700, 200, 3000, tc="tf32")
    assert p["tc"] == 1 and p["kernels"] >= 2 and p["workspace_bytes"] >= 3000 * 200 * 4


@pytest.mark.parametrize("m,k,n", [(1024, 4096, 64), (300, 1000, 256), (512, 776, 272)])
def test_shgemm_tiled_tf32_equals_column_major(shg, m, k, n):
    """SHGEMM-TF32 reading a k-tiled Omega (widened to 32-k FP32 tiles) == the column-major path."""
    g = torch.Generator(device="cuda").manual_seed(m)
    A = torch.randn(m, k, device="cuda", generator=g)
    y_cm = shg.shgemm(A, shg.gen_omega(k, n, seed=6), tc="tf32")
    y_t = shg.shgemm_tiled(A, shg.gen_omega_tiled(k, n, seed=6), n, tune={"tc": "tf32"})
    torch.cuda.synchronize()
    assert torch.equal(y_cm, y_t)


def test_project_tf32_large_k_bars(shg, orc):
    """project(tc='tf32') on an unfolding with K = 2^18 (k-tiled Omega path), sampled rows vs oracle."""
    from oracle import pipelines as opl
    dims = (256, 512, 512)
    T = synth.gaussian(int(np.prod(dims)), 1, seed=21).reshape(dims)
    W = to_np(shg.project(cuda(T), 0, 64, seed=3, tc="tf32"))
    rows = [0, 7, 100, 255]
    A0 = np.ascontiguousarray(opl.unfold(T, 0)[rows])
    check_bars(orc, A0, orc.omega_f16(A0.shape[1], 64, seed=3, stream_id=0), W[rows])
