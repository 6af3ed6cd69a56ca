"""Oracle RandNLA pipelines: Randomized SVD (Alg 1) and RP-HOSVD
(Alg 2), plain numpy on the CPU.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Line 1 of Alg 1 and line 2 of Alg 2 (the
random projection) use the C oracle's naive-FP32 GEMM (``gemm_y32``) or its FP64 GEMM
(``gemm_y64``) with the FP16 Ω of OMEGA_SPEC; QR, SVD and the other products are LAPACK/BLAS
library calls through numpy (the paper uses cuSOLVER/cuBLAS for them).
Residuals are always evaluated in FP64.
"""
from __future__ import annotations

import numpy as np

from . import GAUSSIAN, gemm_y32, gemm_y64, omega_f16


def _qr_pos(Y):
    """Householder QR (LAPACK via numpy) with the R diagonal made non-negative."""
    Q, R = np.linalg.qr(Y)
    d = np.sign(np.diag(R))
    d[d == 0] = 1
    return Q * d[None, :].astype(Q.dtype), R * d[:, None].astype(R.dtype)


def rsvd(A, p: int, s: int = 10, seed: int = 0, precision: str = "f32", dist: int = GAUSSIAN,
         omega_bits=None):
    """Alg 1, p-rank with oversampling s, FP16 Ω.

    precision 'f32': every line in binary32 (the FP32 oracle pipeline the GPU pipeline is
    compared with); 'f64': every line in binary64 (reference for the Halko bound tests).
    Returns dict with U (m x p), S (p), V (n x p), Q, residual ||A - U S V^T||_F / ||A||_F.
    """
    A = np.asarray(A, dtype=np.float32)
    m, n = A.shape
    nhat = p + s
    if omega_bits is None:
        omega_bits = omega_f16(n, nhat, seed=seed, dist=dist, stream_id=0)
    if precision == "f32":
        Y = gemm_y32(A, omega_bits)                              # line 1
        Q, _ = _qr_pos(Y.astype(np.float32))                     # line 2
        B = Q.T.astype(np.float32) @ A                           # line 3 (binary32)
        Uh, S, Vt = np.linalg.svd(B, full_matrices=False)        # line 4
        U = Q @ Uh[:, :p]                                        # line 5
    elif precision == "f64":
        A64 = A.astype(np.float64)
        Y = gemm_y64(A, omega_bits)
        Q, _ = _qr_pos(Y)
        B = Q.T @ A64
        Uh, S, Vt = np.linalg.svd(B, full_matrices=False)
        U = Q @ Uh[:, :p]
    else:
        raise ValueError(precision)
    S = S[:p]
    V = Vt[:p].T
    return {"U": U, "S": S, "V": V, "Q": Q, "Y": Y,
            "residual": reconstruction_error(A, U, S, V)}


def reconstruction_error(A, U, S, V) -> float:
    """||A - U diag(S) V^T||_F / ||A||_F in binary64."""
    A64 = np.asarray(A, dtype=np.float64)
    R = A64 - (np.asarray(U, np.float64) * np.asarray(S, np.float64)[None, :]) @ np.asarray(V, np.float64).T
    return float(np.linalg.norm(R) / np.linalg.norm(A64))


def projection_error(A, Q) -> float:
    """||A - Q Q^T A||_F (Eq 3/4), binary64."""
    A64 = np.asarray(A, dtype=np.float64)
    Q64 = np.asarray(Q, dtype=np.float64)
    return float(np.linalg.norm(A64 - Q64 @ (Q64.T @ A64)))


def halko_bound(sigma, p: int, s: int) -> float:
    """Right side of Eq 4: sqrt(1 + p/(s-1)) * ||Sigma_2||_F."""
    sigma = np.asarray(sigma, dtype=np.float64)
    return float(np.sqrt(1.0 + p / (s - 1.0)) * np.sqrt(np.sum(sigma[p:] ** 2)))


# ----------------------------------------------------------------------------- tensors
def unfold(T, mode: int):
    """Mode-i unfolding A'_(i) in R^{I_i x prod_{k != i} I_k} (Alg 2 line 2);
    column index = C-order linear index over the remaining modes in ascending order."""
    T = np.asarray(T)
    return np.moveaxis(T, mode, 0).reshape(T.shape[mode], -1)


def mode_product(T, M, mode: int):
    """T x_i M with M of shape (I_i, J): contracts M^T . unfold_i(T), mode-i extent -> J
    (SPEC.md:406 orientation; reading c4-19 of SURVEY)."""
    out = np.tensordot(T, M, axes=([mode], [0]))  # contracted mode removed, J appended last
    return np.moveaxis(out, -1, mode)


def rp_hosvd(T, ranks, seed: int = 0, precision: str = "f32", dist: int = GAUSSIAN):
    """Alg 2: for each mode W = A'_(i) Omega_(i), Q_i = QR(W); then
    g = A x_1 Q_1^T ... x_N Q_N^T. Omega_(i) from OMEGA_SPEC with stream_id = i."""
    T = np.asarray(T, dtype=np.float32)
    N = T.ndim
    Qs = []
    for i in range(N):
        Ai = np.ascontiguousarray(unfold(T, i))
        om = omega_f16(Ai.shape[1], ranks[i], seed=seed, dist=dist, stream_id=i)
        W = gemm_y32(Ai, om) if precision == "f32" else gemm_y64(Ai, om)
        Q, _ = _qr_pos(W)
        Qs.append(Q)
    dt = np.float32 if precision == "f32" else np.float64
    g = T.astype(dt)
    for i in range(N):
        g = mode_product(g, Qs[i].astype(dt), i)
    return {"core": g, "Q": Qs, "residual": hosvd_error(T, g, Qs)}


def hosvd_error(T, core, Qs) -> float:
    """||A - g x_1 Q_1 ... x_N Q_N||_F / ||A||_F in binary64."""
    R = np.asarray(core, dtype=np.float64)
    for i, Q in enumerate(Qs):
        R = mode_product(R, np.asarray(Q, np.float64).T, i)
    T64 = np.asarray(T, dtype=np.float64)
    return float(np.linalg.norm(T64 - R) / np.linalg.norm(T64))
