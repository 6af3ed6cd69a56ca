"""Shared helpers for the -m gpu parity tests: the north_star accuracy bars."""
import numpy as np

U32 = 2.0 ** -24


def to_np(t):
    return t.detach().cpu().numpy()


def omega_bits(Om):
    """torch (k, n) float16 column-major view -> numpy (k, n) uint16 bits."""
    return to_np(Om.contiguous()).view(np.uint16)


def check_bars(orc, A, om_bits, Y, rows=None, ratio=2.0, abs_bar=1e-5, slack=1.2):
    """north_star: rel_F(Y_gpu, Y64) <= 2 * rel_F(Y32, Y64) and <= 1e-5 (readings c4-11, c5-3);
    elementwise |Y_gpu - Y64| <= 1.2 [((1/8) k + 3) u |A||Omega| + 2^-36 T|Omega|] (P:594-597 + split
    term, c5-4; T = 1{|a| < 2^-13}: the split's absolute error floor where hi or the scaled lo leave
    the FP16 normal range, DESIGN R22). ratio = inf skips the ratio bar (tiny k)."""
    A = np.asarray(A, dtype=np.float32)
    y64 = orc.gemm_y64(A, om_bits, rows=rows)
    y32 = orc.gemm_y32(A, om_bits, rows=rows)
    Y = np.asarray(Y, dtype=np.float32)
    e_gpu = orc.relative_error(Y, y64)
    e_32 = orc.relative_error(y32, y64)
    k = A.shape[1]
    W = np.abs(orc.f16_bits_as_float(om_bits).astype(np.float64))
    Aabs = np.abs(A if rows is None else A[np.asarray(rows)]).astype(np.float64)
    bound = slack * (((k / 8.0) + 3.0) * U32 * (Aabs @ W) + 2.0 ** -36 * ((Aabs < 2.0 ** -13) @ W))
    err = np.abs(Y.astype(np.float64) - y64)
    worst = float(np.max(err / np.maximum(bound, 1e-300)))
    assert e_gpu <= abs_bar, (e_gpu, e_32)
    assert worst <= 1.0, worst
    # the ratio bar compares two Frobenius errors, i.e. two sums of independent roundings: with fewer
    # than 64 outputs it is a high-variance statistic (a single naive FP32 dot product can round to
    # its exact value by chance), so it applies from 64 outputs on (DESIGN R26); the elementwise bar
    # above always applies
    if ratio != float("inf") and Y.size >= 64:
        assert e_gpu <= ratio * e_32, (e_gpu, e_32)
    return e_gpu, e_32, worst
