"""Pins for the oracle's Ω generator (OMEGA_SPEC.md).

Each test checks the oracle against something other than itself: published KAT vectors,
libm/numpy transcendentals over every input code, numpy's FP16 rounding, and distribution
statistics of N(0,1) and of Eq 7's sparse matrices.
"""
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_kat(orc):
    """Random123 philox4x32_10 known-answer vectors (tests/golden/philox_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(t, 16) for t in line.split()]
        assert orc.philox4x32_10(w[0:4], w[4:6]) == tuple(w[6:10])
        n += 1
    assert n == 3


def test_ln_spec_all_inputs(orc):
    """ln_spec(na) vs binary64 log(na 2^-24) for every na in [1, 2^24] (OMEGA_SPEC §3.1)."""
    na = np.arange(1, (1 << 24) + 1, dtype=np.uint32)
    got = orc.ln_spec_batch(na).astype(np.float64)
    ref = np.log(na.astype(np.float64) * 2.0 ** -24)
    err = np.abs(got - ref)
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    # one rounding of L plus < 1e-7 from LN2/polynomial truncation
    assert np.all(err <= ulp + 1.0e-7), float(np.max(err - ulp))
    assert got[-1] == 0.0  # u = 1 -> L = 0 exactly
    assert np.all(got <= 0.0)


def test_sincos_spec_all_angle_codes(orc):
    """cos/sin of theta = 2 pi code 2^-24 for all 2^24 codes vs binary64 libm (OMEGA_SPEC §3.2)."""
    code = np.arange(1 << 24, dtype=np.uint32)
    c, s = orc.sincos_spec_batch(code << np.uint32(8))
    th = 2.0 * math.pi * code.astype(np.float64) * 2.0 ** -24
    ec = np.max(np.abs(c.astype(np.float64) - np.cos(th)))
    es = np.max(np.abs(s.astype(np.float64) - np.sin(th)))
    assert ec < 2.0e-7 and es < 2.0e-7, (ec, es)
    # low 8 bits of xb never matter
    c2, s2 = orc.sincos_spec_batch((code[:4096] << np.uint32(8)) | np.uint32(0xAB))
    assert np.array_equal(c2, c[:4096]) and np.array_equal(s2, s[:4096])


def test_radius_extremes(orc):
    assert orc.radius_spec(0xFFFFFFFF) == 0.0          # na = 2^24 -> u = 1
    r_max = orc.radius_spec(0x000000FF)                # na = 1 -> u = 2^-24
    assert abs(r_max - math.sqrt(2 * 24 * math.log(2))) < 1e-5


def test_radius_spec_all_codes(orc):
    """r = sqrt(-2 ln u), u = ((xa >> 8) + 1) 2^-24, for every 24-bit code vs binary64 libm
    (OMEGA_SPEC §3.1, Box-Muller radius of the Gaussian Omega); the batch form
    agrees with the scalar one and ignores the low 8 bits."""
    code = np.arange(1 << 24, dtype=np.uint32)
    r = orc.radius_spec_batch(code << np.uint32(8)).astype(np.float64)
    ref = np.sqrt(-2.0 * np.log((code.astype(np.float64) + 1.0) * 2.0 ** -24))
    # ln error <= ulp(L) + 1e-7 (test_ln_spec_all_inputs); sqrt halves the relative error, adds 1 rounding
    dL = np.spacing(np.float32(1.0)) * np.maximum(ref * ref / 2.0, 1e-30) + 1.0e-7
    bound = dL / np.maximum(ref, 1e-30) + np.spacing(ref.astype(np.float32)).astype(np.float64)
    ok = ref > 0
    assert np.all(np.abs(r - ref)[ok] <= bound[ok] * 1.01), float(np.max((np.abs(r - ref) - bound)[ok]))
    assert r[-1] == 0.0
    for i in (0, 1, 77, 1 << 23, (1 << 24) - 2):
        assert r[i] == orc.radius_spec(int(i) << 8 | 0x5A)


def _gauss_sample(orc, count, columns=4, seed=12345, stream=0):
    per = count // columns
    return np.concatenate([orc.gauss_column_f32(seed, stream, j, 0, per) for j in range(columns)])


def test_gaussian_moments_and_ks(orc):
    """N(0,1): mean, variance, kurtosis and a KS test on 2^22 draws."""
    from scipy import stats
    z = _gauss_sample(orc, 1 << 22).astype(np.float64)
    N = z.size
    assert abs(z.mean()) < 5.0 / math.sqrt(N)
    assert abs(z.var() - 1.0) < 5.0 * math.sqrt(2.0 / N)
    kurt = np.mean(z ** 4) / z.var() ** 2
    assert abs(kurt - 3.0) < 5.0 * math.sqrt(24.0 / N)
    D = stats.kstest(z, "norm").statistic
    assert D < 2.0 / math.sqrt(N), D
    # symmetry
    assert abs(np.mean(z > 0) - 0.5) < 5 * 0.5 / math.sqrt(N)


def test_gaussian_pairs_uncorrelated(orc):
    z = orc.gauss_column_f32(7, 0, 3, 0, 1 << 20).astype(np.float64)
    N = z.size // 2
    for lag in (1, 2, 3, 4):
        r = np.corrcoef(z[:-lag], z[lag:])[0, 1]
        assert abs(r) < 5.0 / math.sqrt(N), (lag, r)


def test_omega_is_rn_f16_of_z(orc):
    """Ω = RN_f16(z): compared with numpy's own float32->float16 rounding."""
    k, n = 4096, 6
    om = orc.omega_f16(k, n, seed=99, stream_id=5)
    for j in range(n):
        z = orc.gauss_column_f32(99, 5, j, 0, k)
        ref = z.astype(np.float16).view(np.uint16)
        assert np.array_equal(om[:, j], ref)


def test_omega_fp16_subnormal_rate(orc):
    """FP16-subnormal-or-zero outputs occur with P(|z| < 2^-14) ~ 2 phi(0) 2^-14 = 4.87e-5
    (reading c4-20 of SURVEY; PAPER.md:237-271 studies these rates)."""
    z = _gauss_sample(orc, 1 << 24, columns=8, seed=3)
    h = orc.f32_to_f16_batch(z)
    frac_sub = np.mean((h & 0x7C00) == 0)
    p = 2.0 / math.sqrt(2 * math.pi) * 2.0 ** -14
    sd = math.sqrt(p / z.size)
    assert abs(frac_sub - p) < 5 * sd, (frac_sub, p)


def test_omega_addressing_independent_of_shape(orc):
    """Ω[i][j] depends only on (seed, stream, i, j) (OMEGA_SPEC §2)."""
    big = orc.omega_f16(1000, 40, seed=2024, stream_id=1)
    small = orc.omega_f16(123, 7, seed=2024, stream_id=1)
    assert np.array_equal(big[:123, :7], small)
    sub = orc.omega_f16(300, 40, seed=2024, stream_id=1, row0=501)
    assert np.array_equal(big[501:801], sub)
    other_stream = orc.omega_f16(123, 7, seed=2024, stream_id=2)
    assert not np.array_equal(other_stream, small)
    other_seed = orc.omega_f16(123, 7, seed=2025, stream_id=1)
    assert not np.array_equal(other_seed, small)
    # 64-bit seed and q high word reach the counter
    seed = (5 << 32) | 7                                   # key = (7, 5)
    x = orc.philox4x32_10([1, 2, 9, 0], [7, 5])            # row 6 -> q = 1, word 2; stream 9
    assert orc.omega_element(seed, 9, 1, 10, 6, 2) == (0xBC00 if x[2] >> 31 else 0x3C00)
    hi_row = (1 << 34) + 5
    x = orc.philox4x32_10([(hi_row >> 2) & 0xFFFFFFFF, 3, 0, hi_row >> 34], [0, 0])
    assert orc.omega_element(0, 0, 1, 10, hi_row, 3) == (0xBC00 if x[1] >> 31 else 0x3C00)


def test_rademacher(orc):
    """Eq 7 with s = 1: entries +-1 with probability 1/2 each, no zeros."""
    om = orc.omega_f16(4096, 64, seed=1, dist=orc.RADEMACHER)
    vals, counts = np.unique(om, return_counts=True)
    assert set(vals.tolist()) == {0x3C00, 0xBC00}
    N = om.size
    assert abs(counts[0] / N - 0.5) < 5 * 0.5 / math.sqrt(N)
    # value rule: sign bit of the Philox word
    x = orc.philox4x32_10([0, 0, 0, 0], [1, 0])
    assert om[0, 0] == (0xBC00 if x[0] >> 31 else 0x3C00)
    assert om[3, 0] == (0xBC00 if x[3] >> 31 else 0x3C00)


@pytest.mark.parametrize("dist,k,s", [(2, 4096, 3.0), (3, 10000, 100.0)])
def test_sparse_sign(orc, dist, k, s):
    """Eq 7 without the sqrt(s) factor: P(+1)=P(-1)=1/2s."""
    om = orc.omega_f16(k, 64, seed=5, dist=dist, k_total=k)
    N = om.size
    nz = np.mean(om != 0)
    p = 1.0 / s
    assert abs(nz - p) < 5 * math.sqrt(p * (1 - p) / N)
    pos = np.mean(om == 0x3C00)
    assert abs(pos - p / 2) < 5 * math.sqrt(p / 2 / N)
    assert set(np.unique(om).tolist()) <= {0, 0x3C00, 0xBC00}
    T = orc.sparse_threshold(dist, k)
    assert T == math.floor(2 ** 31 / s)


@pytest.mark.parametrize("stream_id", [0, 1, 2])
def test_square_blocks_full_rank(orc, stream_id):
    """SURVEY c6 / S:317: k x k blocks of the FP16 Gaussian Omega are of full rank for k <= 64 (a
    generator with a stuck counter field or a repeated column would produce rank-deficient blocks)."""
    for k in (1, 2, 3, 4, 8, 16, 32, 64):
        for seed in (0, 7, 12345):
            om = orc.f16_bits_as_float(orc.omega_f16(k, k, seed=seed, stream_id=stream_id)).astype(np.float64)
            assert np.linalg.matrix_rank(om) == k, (k, seed, stream_id)
