"""GPU parity tests for TCEC-SGEMM (Eqs 5-9): C = A.B with
FP32 A and B on the FP16 tensor cores, through the C ABI (`tcec_sgemm_ex`), against the oracle's
FP32 x FP32 GEMMs (oracle.gemm_y64_f32b / gemm_y32_f32b / gemm_ytcec64):
  * exact cases bit-exact (small-integer A and B; identity operands reproduce the split's
    reconstruction RN_f32(hi + lo 2^-11) of the other operand, Eq 16);
  * otherwise the north_star bars of DESIGN.md §3 with B in place of Omega:
    rel_F(C, C64) <= 2 rel_F(C32, C64) and <= 1e-5, and elementwise
    |C - C64| <= 1.2 ((k/8) + 9) u |A||B| (DESIGN R20: +6u over SHGEMM's bar for B's split and
    Eq 9's dropped dA_low dB_low term);
  * every operand layout, single CTAs / CTA pairs, split-K, ragged tails, the CUDA-core fallback,
    and the RSVD line-3 product B^T = A^T Q at the cfg2 size on sampled rows."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24


@pytest.fixture(scope="module")
def shg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_04612_b200 import _build
    _build.build()
    import paper_2304_04612_b200 as m
    assert m.device_supported(), "device is not sm_100"
    return m


def _dev(a, layout, k_dim):
    """numpy 2-D -> cuda tensor with the requested contiguous dimension (0 = k contiguous)."""
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if layout == 0:     # K-major: the k dimension contiguous
        return t if k_dim == 1 else t.t().contiguous().t()
    return t.t().contiguous().t() if k_dim == 1 else t


def run(shg, A, B, la=0, lb=0, tune=None):
    C = shg.tcec_sgemm(_dev(A, la, 1), _dev(B, lb, 0), tune=tune)
    torch.cuda.synchronize()
    return C.cpu().numpy()


def check_bars(orc, A, B, C, rows=None, ratio=2.0, abs_bar=1e-5, slack=1.2):
    A = np.asarray(A, dtype=np.float32)
    B = np.asarray(B, dtype=np.float32)
    y64 = orc.gemm_y64_f32b(A, B, rows=rows)
    y32 = orc.gemm_y32_f32b(A, B, rows=rows)
    e_gpu = orc.relative_error(C, y64)
    e_32 = orc.relative_error(y32, y64)
    Aabs = np.abs(A if rows is None else A[np.asarray(rows)]).astype(np.float64)
    Babs = np.abs(B).astype(np.float64)
    # + the split floor of DESIGN R22 for either operand (2^-35: representation + dropped term)
    bound = slack * (((A.shape[1] / 8.0) + 9.0) * U32 * (Aabs @ Babs) +
                     2.0 ** -35 * ((Aabs < 2.0 ** -13) @ Babs + Aabs @ (Babs < 2.0 ** -13)))
    worst = float(np.max(np.abs(C.astype(np.float64) - y64) / np.maximum(bound, 1e-300)))
    assert e_gpu <= abs_bar, (e_gpu, e_32)
    assert e_gpu <= ratio * e_32, (e_gpu, e_32)
    assert worst <= 1.0, worst
    return e_gpu, e_32, worst


@pytest.mark.parametrize("m,k,n", [(300, 640, 96), (512, 512, 272), (128, 1000, 40), (77, 200, 130)])
@pytest.mark.parametrize("la,lb", [(0, 0), (1, 1), (0, 1), (1, 0)])
def test_exact_integer_case_bitwise(shg, orc, m, k, n, la, lb):
    """|a|, |b| <= 8 integers: FP16-exact (lo = 0), all partial sums exact in FP32 -> C == A.B."""
    rng = np.random.default_rng(m + k + n)
    A = rng.integers(-8, 9, (m, k)).astype(np.float32)
    B = rng.integers(-8, 9, (k, n)).astype(np.float32)
    C = run(shg, A, B, la, lb)
    np.testing.assert_array_equal(C, (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32))


def _reconstruct(orc, x):
    hi, lo = orc.split(x.astype(np.float32))
    h = orc.f16_bits_as_float(hi).astype(np.float32).reshape(x.shape)
    l = orc.f16_bits_as_float(lo).astype(np.float32).reshape(x.shape)
    return (h.astype(np.float64) + l.astype(np.float64) * 2.0 ** -11).astype(np.float32)


def test_identity_b_reconstructs_split_of_a(shg, orc):
    """B = I: each C element is one product, so C == RN_f32(A_low + dA_low 2^-11) bit for bit."""
    rng = np.random.default_rng(7)
    A = (rng.standard_normal((384, 256)) * np.exp(rng.uniform(-6, 6, (384, 256)))).astype(np.float32)
    C = run(shg, A, np.eye(256, dtype=np.float32))
    np.testing.assert_array_equal(C, _reconstruct(orc, A))


def test_identity_a_reconstructs_split_of_b(shg, orc):
    """A = I: C == RN_f32(B_low + dB_low 2^-11) — checks the B-side split and the A_low.dB_low term."""
    rng = np.random.default_rng(8)
    B = (rng.standard_normal((192, 160)) * np.exp(rng.uniform(-6, 6, (192, 160)))).astype(np.float32)
    for lb in (0, 1):
        C = run(shg, np.eye(192, dtype=np.float32), B, 0, lb)
        np.testing.assert_array_equal(C, _reconstruct(orc, B))


@pytest.mark.parametrize("m,k,n", [(512, 512, 32), (1000, 2048, 272), (256, 4096, 64), (130, 777, 200),
                                   (4096, 256, 256), (64, 16384, 64), (700, 1000, 300), (128, 512, 272),
                                   (640, 333, 288)])
@pytest.mark.parametrize("la,lb", [(0, 0), (1, 1)])
def test_bars_gaussian(shg, orc, m, k, n, la, lb):
    rng = np.random.default_rng(m * 7 + n)
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    check_bars(orc, A, B, run(shg, A, B, la, lb))


def test_bars_orthonormal_q(shg, orc):
    """The RSVD line-3 operand: Q with orthonormal columns (entries ~ 1/sqrt(k)) against a
    matrix with a decaying spectrum, as B^T = A^T Q (A MN-major, Q N-major)."""
    import synth
    s = synth.spectrum("exp", 1024, 64, 1e-2)
    A = synth.spectrum_matrix(s, seed=3).astype(np.float32)
    Q, _ = np.linalg.qr(np.random.default_rng(4).standard_normal((1024, 80)))
    Q = Q.astype(np.float32)
    Bt = shg.tcec_sgemm(torch.from_numpy(A).cuda().t(), torch.from_numpy(Q).cuda())
    torch.cuda.synchronize()
    check_bars(orc, np.ascontiguousarray(A.T), Q, Bt.cpu().numpy())


@pytest.mark.parametrize("tune", [{"split_k": 3}, {"pair": 2, "bn": 64}, {"pair": 1, "bn": 128}, {"bn": 32},
                                  {"max_ctas": 6}, {"pair": 2, "bn": 128}, {"bn": 256}])
def test_tunables(shg, orc, tune):
    rng = np.random.default_rng(11)
    A = rng.standard_normal((600, 1536)).astype(np.float32)
    B = rng.uniform(-1, 1, (1536, 250)).astype(np.float32)
    check_bars(orc, A, B, run(shg, A, B, tune=tune))


def test_plans(shg):
    p = shg.tcec_plan(16384, 272, 16384)
    assert p["path"] == 0 and p["tc"] == 2 and p["cta_pair"] == 1 and p["bn"] == 272 and p["n_tiles"] == 1
    p1 = shg.tcec_plan(100, 200, 512)          # one row block: single CTAs, BN capped at 128
    assert p1["cta_pair"] == 0 and p1["bn"] <= 128
    with pytest.raises(shg.SHGError):
        shg.tcec_plan(100, 200, 512, tune={"bn": 256, "pair": 2})


def test_fallback_misaligned(shg, orc):
    """lda % 4 != 0 takes the CUDA-core fallback; same bars."""
    rng = np.random.default_rng(12)
    A = rng.standard_normal((100, 301)).astype(np.float32)
    B = rng.standard_normal((301, 37)).astype(np.float32)
    At = torch.from_numpy(A).cuda()
    assert At.stride(0) % 4 != 0
    C = shg.tcec_sgemm(At, torch.from_numpy(B).cuda())
    torch.cuda.synchronize()
    check_bars(orc, A, B, C.cpu().numpy())
    Cs = run(shg, A, B, tune={"force_simt": 1})
    check_bars(orc, A, B, Cs)


def test_edge_sizes(shg):
    A = torch.randn(5, 0, device="cuda")
    B = torch.randn(0, 7, device="cuda")
    C = shg.tcec_sgemm(A, B)
    torch.cuda.synchronize()
    assert torch.count_nonzero(C) == 0 and C.shape == (5, 7)
    C = shg.tcec_sgemm(torch.randn(0, 9, device="cuda"), torch.randn(9, 4, device="cuda"))
    assert C.shape == (0, 4)


def test_deterministic(shg):
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(2000, 3000, device="cuda", generator=g)
    B = torch.randn(3000, 200, device="cuda", generator=g)
    C1 = shg.tcec_sgemm(A, B)
    C2 = shg.tcec_sgemm(A, B)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)


def test_rsvd_line3_full_size_sampled(shg, orc):
    """cfg2 (16384^2, n = 272): B^T = A^T Q with A read in place (MN-major); 192 sampled rows of
    B^T (= columns of A) checked against the oracle."""
    import synth
    N, nh = 16384, 272
    A = synth.spectrum_matrix_torch(synth.spectrum("exp", N, 256, 1e-2), seed=1)
    g = torch.Generator(device="cuda").manual_seed(5)
    Q, _ = torch.linalg.qr(torch.randn(N, nh, device="cuda", generator=g))
    Bt = shg.tcec_sgemm(A.t(), Q)
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(6).choice(N, 192, replace=False))
    rows[0], rows[-1] = 0, N - 1
    cols = torch.from_numpy(rows).cuda()
    At_rows = A[:, cols].t().contiguous().cpu().numpy()
    check_bars(orc, At_rows, Q.cpu().numpy(), Bt[cols].cpu().numpy())
