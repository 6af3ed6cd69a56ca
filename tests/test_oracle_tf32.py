"""Pins for the oracle's SHGEMM-TF32 pieces (Eqs 14-15 with toLow = TF32):
the FP32 -> TF32 RN conversion (exhaustively, against F16C by exponent scaling), the TF32 split
(worked examples, exact-rational nearest-value check, inequalities), and Eq 16 in FP64."""
import ctypes
import os
from fractions import Fraction

import numpy as np
import pytest

from test_oracle_f16_split import f16c  # noqa: F401  (shared helper-library fixture)

HERE = os.path.dirname(__file__)
GOLDEN = os.path.join(HERE, "golden")


def test_tf32_exhaustive_vs_f16c_scaling(f16c):  # noqa: F811
    """All 2^32 FP32 patterns: orc_f32_to_tf32_rn == RN_f16(y) * 2^e (F16C) for normal x = y 2^e,
    == integer RN at quantum 2^-136 for subnormals; inf/zero kept, NaN stays NaN."""
    f16c.tf32_mismatches.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32)]
    f16c.tf32_mismatches.restype = ctypes.c_uint64
    first = ctypes.c_uint32(0)
    bad = f16c.tf32_mismatches(0, 1 << 32, ctypes.byref(first))
    assert bad == 0, hex(first.value)


def test_split_tf32_golden(orc):
    """Hand-derived worked examples, tests/golden/split_tf32_examples.txt (derivations inside)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "split_tf32_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        a_bits, hi_bits, lo_bits = (int(t, 16) for t in line.split()[:3])
        a = np.array([a_bits], dtype=np.uint32).view(np.float32)
        hi, lo = orc.split_tf32(a)
        assert (int(hi[0]), int(lo[0])) == (hi_bits, lo_bits), line
        n += 1
    assert n == 11


def _nearest_11bit(x: Fraction) -> Fraction:
    """RN ties-to-even of a positive rational to 11 significant bits (unbounded exponent)."""
    e = x.numerator.bit_length() - x.denominator.bit_length()
    while Fraction(2) ** e > x:
        e -= 1
    while Fraction(2) ** (e + 1) <= x:
        e += 1
    q = Fraction(2) ** (e - 10)                  # ulp of an 11-bit significand in [2^e, 2^(e+1))
    t = x / q
    fl = t.numerator // t.denominator
    rem = t - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return fl * q


def test_tf32_rounding_is_nearest_11_bit_value(orc):
    """Exact-rational check on random normal values: hi is the nearest value with an 11-bit
    significand (ties to even), independent of any float arithmetic."""
    rng = np.random.default_rng(7)
    bits = rng.integers(0x00800000, 0x7F000000, size=4000, dtype=np.uint32)
    a = bits.view(np.float32)
    hi, _ = orc.split_tf32(a)
    for x, h in zip(a, hi):
        ref = _nearest_11bit(Fraction(float(x)))
        got = Fraction(float(np.array([h], dtype=np.uint32).view(np.float32)[0]))
        assert got == ref, (float(x), float(got), float(ref))


def test_split_tf32_matches_fp16_split_in_fp16_normal_range(orc):
    """TF32 and FP16 share the 10-bit fraction: inside the FP16 normal range the two splits give
    the same hi value, and the same lo wherever the scaled residual is FP16-normal."""
    rng = np.random.default_rng(3)
    N = 1 << 18
    a = (np.exp2(rng.uniform(-13.9, 15.9, N)) * rng.choice([-1.0, 1.0], N)).astype(np.float32)
    a = a[np.abs(a) < 65504]
    h16, l16 = orc.split(a)
    h32, l32 = orc.split_tf32(a)
    hf16 = h16.view(np.float16).astype(np.float32)
    lf16 = l16.view(np.float16).astype(np.float32)
    assert np.array_equal(hf16, h32.view(np.float32))
    normal = np.abs(l32.view(np.float32)) >= 2.0 ** -14   # residual itself FP16-normal
    assert normal.mean() > 0.9
    assert np.array_equal(lf16[normal], l32.view(np.float32)[normal])


def test_split_tf32_inequalities_full_exponent_range(orc):
    """Over the whole FP32 exponent range: low 13 bits of hi and lo are zero,
    |a - (hi + lo 2^-11)| <= 1 ulp_f32(a), zero in ~75% of cases (the 0.25-bit loss of P:572)."""
    rng = np.random.default_rng(4)
    N = 1 << 20
    a = (np.exp2(rng.uniform(-110, 126.9, N)) * rng.choice([-1.0, 1.0], N)).astype(np.float32)
    hi, lo = orc.split_tf32(a)
    assert np.all((hi & 0x1FFF) == 0) and np.all((lo & 0x1FFF) == 0)
    hf = hi.view(np.float32).astype(np.float64)
    lf = lo.view(np.float32).astype(np.float64) * 2.0 ** -11
    a64 = a.astype(np.float64)
    u = 2.0 ** -11
    assert np.all(np.abs(hf) <= (1 + u) * np.abs(a64))
    assert np.all(np.abs(lf) <= u * np.abs(a64))
    delta = a64 - (hf + lf)
    assert np.all(np.abs(delta) <= np.spacing(np.abs(a)).astype(np.float64))
    frac = np.mean(delta != 0)
    assert 0.22 < frac < 0.28, frac


def test_split_tf32_exact_for_tf32_values_and_nan(orc):
    rng = np.random.default_rng(5)
    bits = rng.integers(0, 1 << 32, size=1 << 16, dtype=np.uint64).astype(np.uint32) & ~np.uint32(0x1FFF)
    bits = bits[(bits & 0x7F800000) != 0x7F800000]
    a = bits.view(np.float32)
    hi, lo = orc.split_tf32(a)
    assert np.array_equal(hi, bits)
    assert np.all((lo & 0x7FFFFFFF) == 0)
    hi, lo = orc.split_tf32(np.array([np.nan, np.inf, -np.inf], dtype=np.float32))
    assert (hi[0] & 0x7FFFFFFF) > 0x7F800000
    assert hi[1] == 0x7F800000 and hi[2] == 0xFF800000


def test_ysplit64_tf32(orc):
    """Eq 16 with the TF32 split: equals the FP16-split result for FP16-range A whose lo parts are
    all FP16-normal, and stays finite and FP32-accurate where FP16 overflows (A_Cauchy)."""
    rng = np.random.default_rng(6)
    k, n = 300, 12
    om = orc.omega_f16(k, n, seed=2)
    A = rng.uniform(1.0, 2.0, (20, k)).astype(np.float32)       # lo parts are >= 2^-14 or 0
    np.testing.assert_array_equal(orc.gemm_ysplit64_tf32(A, om), orc.gemm_ysplit64(A, om))
    B = (rng.standard_normal((20, k)) * 1e6).astype(np.float32)  # |a| >> 65504
    y64 = orc.gemm_y64(B, om)
    yt = orc.gemm_ysplit64_tf32(B, om)
    assert np.all(np.isfinite(yt))
    assert not np.all(np.isfinite(orc.gemm_ysplit64(B, om)))
    assert orc.relative_error(yt, y64) < 2.0 ** -22
