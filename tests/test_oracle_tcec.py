"""Pins for the oracle's FP32 x FP32 GEMMs and TCEC-SGEMM (Eqs 5-9), used by the
NEXT-2 row (FP32-accurate tensor-core GEMM for the pipelines' other products)."""
from fractions import Fraction

import numpy as np


def test_f32b_gemms_equal_the_pinned_fp16_omega_gemms(orc):
    """With an FP16-representable B the FP32-B GEMMs must reproduce the already pinned FP16-Omega
    GEMMs bit for bit (same operation order)."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((37, 300)).astype(np.float32)
    om = orc.omega_f16(300, 11, seed=5)
    B = orc.f16_bits_as_float(om)
    np.testing.assert_array_equal(orc.gemm_y64_f32b(A, B), orc.gemm_y64(A, om))
    np.testing.assert_array_equal(orc.gemm_y32_f32b(A, B), orc.gemm_y32(A, om))


def test_y64_f32b_brute_force(orc):
    """Exact rational sum vs the FP64 result within the sequential-summation bound."""
    rng = np.random.default_rng(2)
    A = rng.standard_normal((3, 40)).astype(np.float32)
    B = rng.standard_normal((40, 4)).astype(np.float32)
    Y = orc.gemm_y64_f32b(A, B)
    for i in range(3):
        for j in range(4):
            exact = sum(Fraction(float(A[i, l])) * Fraction(float(B[l, j])) for l in range(40))
            bound = 40 * 2.0 ** -53 * sum(abs(float(A[i, l]) * float(B[l, j])) for l in range(40))
            assert abs(Fraction(Y[i, j]) - exact) <= Fraction(bound)


def test_tcec_exact_for_fp16_operands(orc):
    """lo == 0 for FP16-representable A and B: Eq 9 reduces to A_low B_low == the exact product."""
    rng = np.random.default_rng(3)
    A = rng.integers(-8, 9, (50, 256)).astype(np.float32)
    B = rng.integers(-8, 9, (256, 20)).astype(np.float32)
    np.testing.assert_array_equal(orc.gemm_ytcec64(A, B), A.astype(np.float64) @ B.astype(np.float64))


def test_tcec_transpose_symmetry(orc):
    """Eq 9 is symmetric in its operands: (A B)^T computed as B^T A^T gives the same terms, so the
    result is bit-identical — fails if a correction term is dropped or the wrong lo is used."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((23, 130)).astype(np.float32)
    B = (rng.standard_normal((130, 17)) * 3.0).astype(np.float32)
    np.testing.assert_array_equal(orc.gemm_ytcec64(A, B).T, orc.gemm_ytcec64(B.T, A.T))


def test_tcec_error_bound_and_both_corrections_matter(orc):
    """Per product Eq 9 errs by the two split representation errors (<= 1 FP32 ulp each,
    <= 2u|a|, 2u|b|) plus the dropped 2^-22 dA_low dB_low (<= u16^2 |a||b| = 4u|a||b|), so
    |Y_tcec - Y64| <= 8.01u sum_l |a||b| (u = 2^-24) in the worst case (DESIGN R20); on random
    data of length 512 it is well under 3u. Dropping either correction term costs ~2^-12 relative."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((64, 512)).astype(np.float32)
    B = rng.standard_normal((512, 32)).astype(np.float32)
    y64 = orc.gemm_y64_f32b(A, B)
    yt = orc.gemm_ytcec64(A, B)
    absprod = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
    assert np.all(np.abs(yt - y64) <= 3 * 2.0 ** -24 * absprod)
    # short products do not average: the worst case needs the full 8u (k = 4, fuzz case 1567 of
    # tests/test_gpu_fuzz.py reaches 4.7u); 20000 random 1- to 4-term rows stay within 8.01u
    for kk in (1, 2, 4):
        A2 = (rng.standard_normal((5000, kk)) * np.exp(rng.uniform(-3, 3, (5000, kk)))).astype(np.float32)
        B2 = (rng.standard_normal((kk, 8)) * np.exp(rng.uniform(-3, 3, (kk, 8)))).astype(np.float32)
        ab = np.abs(A2).astype(np.float64) @ np.abs(B2).astype(np.float64)
        err = np.abs(orc.gemm_ytcec64(A2, B2) - orc.gemm_y64_f32b(A2, B2))
        assert np.all(err <= 8.01 * 2.0 ** -24 * ab)
        if kk == 1:     # one product: the split + dropped-term error alone, which exceeds 3u somewhere
            assert np.max(err / np.maximum(ab, 1e-300)) > 3 * 2.0 ** -24
    assert orc.relative_error(yt, y64) < 2e-7
    # no-correction (A_low B_low only) is far worse: FP16-level
    ha, _ = orc.split(A)
    hb, _ = orc.split(B)
    y_hh = (ha.view(np.float16).astype(np.float64).reshape(A.shape) @
            hb.view(np.float16).astype(np.float64).reshape(B.shape))
    assert orc.relative_error(y_hh, y64) > 1e-4
