"""Pins for the oracle GEMMs: Y64 (Fig 5's C_F64), naive FP32 Y32
 and Eq 16 in FP64 (Y_split64).

Pins: identity / permutation A (exact), exact small-integer arithmetic against numpy's
integer matmul, brute force with Python Fractions on tiny inputs, and the textbook error
bounds of recursive summation (Higham: |fl(x^T y) - x^T y| <= gamma_k |x|^T |y|)."""
from fractions import Fraction

import numpy as np
import pytest

import synth


def _omega_float(orc, bits):
    return orc.f16_bits_as_float(bits).astype(np.float64)


def test_identity_and_permutation(orc):
    k, n = 96, 24
    om = orc.omega_f16(k, n, seed=11)
    W = _omega_float(orc, om)
    I = np.eye(k, dtype=np.float32)
    assert np.array_equal(orc.gemm_y64(I, om), W)
    assert np.array_equal(orc.gemm_y32(I, om).astype(np.float64), W)
    assert np.array_equal(orc.gemm_ysplit64(I, om), W)
    perm = np.random.default_rng(0).permutation(k)
    P = I[perm]
    assert np.array_equal(orc.gemm_y64(P, om), W[perm])
    assert np.array_equal(orc.gemm_y32(P, om).astype(np.float64), W[perm])
    # Omega = identity (via the test hook of SPEC.md:451): Y selects columns of A
    A = synth.gaussian(17, k, 3)
    eye_bits = np.eye(k, n, dtype=np.float32).astype(np.float16).view(np.uint16)
    assert np.array_equal(orc.gemm_y32(A, eye_bits), A[:, :n])


def test_exact_integer_case(orc):
    """|a| <= 8 integers times Rademacher Omega: every partial sum is an integer < 2^24, so Y64,
    Y32 and the exact product coincide (derived from PAPER.md:464-469)."""
    m, k, n = 40, 2048, 33
    A = synth.small_int_matrix(m, k, seed=4)
    om = orc.omega_f16(k, n, seed=8, dist=orc.RADEMACHER)
    exact = A.astype(np.int64) @ _omega_float(orc, om).astype(np.int64)
    assert np.array_equal(orc.gemm_y64(A, om), exact.astype(np.float64))
    assert np.array_equal(orc.gemm_y32(A, om).astype(np.float64), exact.astype(np.float64))


@pytest.mark.parametrize("k", [1, 7, 16, 64])
def test_brute_force_fractions(orc, k):
    m, n = 5, 6
    A = synth.gaussian(m, k, seed=100 + k) * np.float32(3.0)
    om = orc.omega_f16(k, n, seed=k)
    W = _omega_float(orc, om)
    Y64 = orc.gemm_y64(A, om)
    Y32 = orc.gemm_y32(A, om).astype(np.float64)
    for i in range(m):
        for j in range(n):
            ex = sum((Fraction(float(A[i, l])) * Fraction(float(W[l, j])) for l in range(k)), Fraction(0))
            mag = sum(abs(float(A[i, l]) * float(W[l, j])) for l in range(k))
            g64 = k * 2.0 ** -53 / (1 - k * 2.0 ** -53)
            g32 = k * 2.0 ** -24 / (1 - k * 2.0 ** -24)
            assert abs(Fraction(Y64[i, j]) - ex) <= Fraction(g64 * mag)
            assert abs(Fraction(Y32[i, j]) - ex) <= Fraction(g32 * mag)


def test_y32_is_sequential_fma(orc):
    """Y32 accumulates in l order: for k = 2, Y32 = fma(a1, w1, a0 w0) exactly; the reversed
    order differs on a crafted case (so a reordered implementation fails)."""
    A = np.array([[1.0, 2.0 ** -24]], dtype=np.float32)
    A2 = np.array([[2.0 ** -24, 1.0]], dtype=np.float32)
    om = np.array([[1.0], [1.0]], dtype=np.float32).astype(np.float16).view(np.uint16)
    # 1 + 2^-24 ties to 1 in fp32 either way; use 3 terms to expose order
    A3 = np.array([[1.0, 2.0 ** -24, 2.0 ** -24]], dtype=np.float32)
    om3 = np.ones((3, 1), dtype=np.float32).astype(np.float16).view(np.uint16)
    assert orc.gemm_y32(A3, om3)[0, 0] == np.float32(1.0)           # ((1 + e) + e) = 1
    A3r = np.array([[2.0 ** -24, 2.0 ** -24, 1.0]], dtype=np.float32)
    assert orc.gemm_y32(A3r, om3)[0, 0] == np.float32(1.0 + 2.0 ** -23)  # (e + e) + 1
    assert orc.gemm_y32(A, om)[0, 0] == orc.gemm_y32(A2, om)[0, 0]


def test_ysplit64(orc):
    """Eq 16 in FP64: equals Y64 when A is FP16-exact; otherwise differs only by the split
    loss A_delta (|A_delta| <= u_F16^2 |a|)."""
    k, n = 512, 16
    om = orc.omega_f16(k, n, seed=1)
    W = np.abs(_omega_float(orc, om))
    A16 = synth.gaussian(8, k, seed=2).astype(np.float16).astype(np.float32)
    assert np.array_equal(orc.gemm_ysplit64(A16, om), orc.gemm_y64(A16, om))
    A = synth.gaussian(8, k, seed=3)
    d = np.abs(orc.gemm_ysplit64(A, om) - orc.gemm_y64(A, om))
    bound = (2.0 ** -22) * (np.abs(A).astype(np.float64) @ W) + 1e-300
    assert np.all(d <= bound)


def test_sampled_rows_match_full(orc):
    A = synth.uniform(50, 300, seed=9)
    om = orc.omega_f16(300, 12, seed=3)
    rows = np.array([49, 0, 17, 17, 3])
    assert np.array_equal(orc.gemm_y32(A, om, rows=rows), orc.gemm_y32(A, om)[rows])
    assert np.array_equal(orc.gemm_y64(A, om, rows=rows), orc.gemm_y64(A, om)[rows])


def test_relative_error_metric(orc):
    C = np.arange(12.0).reshape(3, 4) + 1
    assert orc.relative_error(C, C) == 0.0
    assert orc.relative_error(2 * C, C) == pytest.approx(1.0)


def test_fig5_shape_error_growth(orc):
    """Naive FP32 error vs FP64 grows with k (S:611 analogue of Fig 5), and stays at the
    binary32 level (<= 1e-5) for k <= 4096 with A ~ N(0,1), B ~ N(0,1)."""
    errs = []
    for k in (64, 1024, 4096):
        A = synth.gaussian(64, k, seed=k)
        om = orc.omega_f16(k, 32, seed=0)
        errs.append(orc.relative_error(orc.gemm_y32(A, om), orc.gemm_y64(A, om)))
    assert errs[0] < errs[2] and max(errs) < 1e-5


def test_synth_rows_counter_based(orc):
    """OMEGA_SPEC §6 synthetic rows: same Philox/Box-Muller as Ω, kept in fp32."""
    r = orc.synth_rows("gauss", 2, 0x100, [0, 5], 16)
    z = orc.gauss_column_f32(2, 0x100, 5, 0, 16)
    assert np.array_equal(r[1], z)
    u = orc.synth_rows("unif", 2, 0x100, [3], 8)[0]
    x = orc.philox4x32_10([1, 3, 0x100, 0], [2, 0])
    assert u[5] == np.float32((x[1] >> 8) * 2.0 ** -24)
    assert np.all((u >= 0) & (u < 1))
