"""Seeded synthetic inputs shaped like the paper's workloads (DESIGN.md §4 "input recipe").

This module is shared by the tests, the oracle side and the GPU side. It holds none of the
method's arithmetic (no Ω generation, no split, no GEMM under test): only test matrices and
tensors, built in binary64 with numpy and rounded once to binary32.

Recipes (PAPER.md citations):
  spectrum()          s_i for A_linear / A_exp, 0-indexed i = 0..N-1
  eckart_young_floor  closed forms P:684-691 (A_linear: s_p sqrt(N-p); A_exp: tail sum)
  haar()              Haar orthogonal via QR of a Gaussian with sign fix
  spectrum_matrix()   U diag(s) V^T (slatms replaced); 'hadamard' factors for N=16384
  alg3_tensor()       Alg 3, padding p, normalised to unit RMS (DESIGN.md reading);
                      alg3_tensor_torch() the same draws evaluated on the GPU (bench's 1024^3 input)
  cauchy_like()       A_Cauchy + one A A^T A step so that |a| > 65504
  gaussian/uniform    A ~ N(0,1) or U(0,1)
"""
from __future__ import annotations

import math

import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def gaussian(m: int, n: int, seed: int) -> np.ndarray:
    return rng(seed).standard_normal((m, n)).astype(np.float32)


def uniform(m: int, n: int, seed: int) -> np.ndarray:
    return rng(seed).random((m, n)).astype(np.float32)


def spectrum(kind: str, N: int, p: int, s_p: float) -> np.ndarray:
    """Singular values of A_linear / A_exp, i = 0..N-1, in binary64."""
    i = np.arange(N, dtype=np.float64)
    if kind == "linear":
        alpha = (1.0 - s_p) / p
        return np.maximum(-alpha * i + 1.0, s_p)
    if kind == "exp":
        alpha = math.log2(1.0 / s_p) / p
        return np.exp2(-alpha * i)
    raise ValueError(kind)


def eckart_young_floor(kind: str, N: int, p: int, s_p: float) -> float:
    """||Sigma_2||_F of Theorem 1 in the closed forms of P:684-691.

    linear: s_p sqrt(N - p). exp: sqrt((s_p^2 - 2^{2qN}) / (1 - 2^{2q})) with
    q = -alpha_e (reading c4-14: the tail is i = p..N-1, geometric with ratio 2^{2q})."""
    if kind == "linear":
        return s_p * math.sqrt(N - p)
    alpha = math.log2(1.0 / s_p) / p
    q = -alpha
    return math.sqrt((s_p ** 2 - 2.0 ** (2 * q * N)) / (1.0 - 2.0 ** (2 * q)))


def haar(n: int, seed: int) -> np.ndarray:
    G = rng(seed).standard_normal((n, n))
    Q, R = np.linalg.qr(G)
    return Q * np.sign(np.diag(R))[None, :]


def _fwht_rows(X: np.ndarray) -> np.ndarray:
    """Unnormalised Walsh-Hadamard transform along axis 0 (Sylvester order), in place copy."""
    X = np.array(X, dtype=np.float64, copy=True)
    n = X.shape[0]
    h = 1
    while h < n:
        Xv = X.reshape(n // (2 * h), 2, h, -1)
        a = Xv[:, 0].copy()
        b = Xv[:, 1]
        Xv[:, 0] = a + b
        Xv[:, 1] = a - b
        h *= 2
    return X


def spectrum_matrix(s: np.ndarray, seed: int, method: str = "haar") -> np.ndarray:
    """A = U diag(s) V^T, square N x N, built in binary64, rounded to binary32.

    method 'haar': U, V Haar (QR of Gaussians). method 'hadamard': U = P1 (H/sqrt N) D1,
    V = P2 (H/sqrt N) D2 with random signs D and permutations P — orthogonal, O(N^2 log N).
    V^T Omega is again Gaussian for Gaussian Omega, so the projection error depends only on s
    (SURVEY §8(d) cfg2 substitution, in the spirit of SPEC.md:566)."""
    N = s.shape[0]
    if method == "haar":
        U = haar(N, seed)
        V = haar(N, seed + 1)
        return ((U * s[None, :]) @ V.T).astype(np.float32)
    if method != "hadamard":
        raise ValueError(method)
    assert N & (N - 1) == 0, "hadamard construction needs N = 2^t"
    g = rng(seed)
    d1 = g.choice([-1.0, 1.0], N)
    d2 = g.choice([-1.0, 1.0], N)
    p1 = g.permutation(N)
    p2 = g.permutation(N)
    # V^T = D2 (H/sqrtN) P2^T ; M = diag(s) V^T : row t = s_t d2_t (H row t) permuted columns
    E = np.zeros((N, N))
    E[np.arange(N), np.arange(N)] = s * d2
    M = _fwht_rows(E) / math.sqrt(N)         # = (H/sqrtN) diag(s d2)  (H symmetric)
    M = M.T                                  # = diag(s d2) (H/sqrtN) = diag(s) D2 H/sqrtN
    M = M[:, np.argsort(p2)]                 # right-multiply by P2^T
    X = d1[:, None] * M                      # D1 M
    A = _fwht_rows(X) / math.sqrt(N)         # (H/sqrtN) D1 M
    A = A[np.argsort(p1)]                    # left-multiply by P1
    return A.astype(np.float32)


def mode_product64(T, M, mode):
    out = np.tensordot(T, M, axes=([mode], [0]))
    return np.moveaxis(out, -1, mode)


def alg3_tensor(dims, ranks, pad: int, seed: int, noise: float = 0.0) -> np.ndarray:
    """Alg 3: G ~ U(-1,1)^{J_1..J_N}; for each mode Omega_(i) =
    Omega_alpha (J_i x (J_i - pad)) . Omega_beta ((J_i - pad) x I_i), both U(-1,1);
    G <- G x_i Omega_(i). Multilinear rank J_i - pad. Normalised to unit RMS; optional
    additive noise eta * N(0,1) (reading c4-18)."""
    g = rng(seed)
    G = g.uniform(-1.0, 1.0, size=tuple(ranks))
    for i, (I, J) in enumerate(zip(dims, ranks)):
        Oa = g.uniform(-1.0, 1.0, size=(J, J - pad))
        Ob = g.uniform(-1.0, 1.0, size=(J - pad, I))
        G = mode_product64(G, Oa @ Ob, i)
    G = G / math.sqrt(np.mean(G * G))
    if noise:
        G = G + noise * g.standard_normal(G.shape)
    return G.astype(np.float32)


def alg3_tensor_torch(dims, ranks, pad: int, seed: int, device="cuda", noise: float = 0.0):
    """alg3_tensor's construction (same random draws) evaluated with torch in FP64 on `device`, FP32
    result — for the 1024^3 RP-HOSVD input of the bench (the numpy version takes minutes). noise > 0
    adds noise * N(0,1) from torch's generator seeded with `seed` (the noisy variant of reading c4-18;
    NOT the numpy variant's draws: both sides of a parity test must use this one tensor)."""
    import torch
    g = rng(seed)
    G = torch.as_tensor(g.uniform(-1.0, 1.0, size=tuple(ranks)), dtype=torch.float64, device=device)
    for i, (I, J) in enumerate(zip(dims, ranks)):
        Oa = g.uniform(-1.0, 1.0, size=(J, J - pad))
        Ob = g.uniform(-1.0, 1.0, size=(J - pad, I))
        M = torch.as_tensor(Oa @ Ob, dtype=torch.float64, device=device)
        G = torch.movedim(torch.tensordot(G, M, dims=([i], [0])), -1, i)
    G = G / torch.sqrt(torch.mean(G * G))
    if noise:
        gen = torch.Generator(device=device).manual_seed(seed)
        G = G.float()
        G.add_(torch.randn(G.shape, generator=gen, device=device, dtype=torch.float32), alpha=noise)
        return G
    return G.float()


def cauchy_like(N: int, seed: int) -> np.ndarray:
    """A_Cauchy: 1/(|x_i - y_j| + gamma), x, y ~ U(-1e-3, 1e-3),
    gamma = 1e-3, followed by one A A^T A step; entries then exceed the FP16 range (65504)."""
    g = rng(seed)
    x = g.uniform(-1e-3, 1e-3, N)
    y = g.uniform(-1e-3, 1e-3, N)
    A = 1.0 / (np.abs(x[:, None] - y[None, :]) + 1e-3)
    A = A @ (A.T @ A) / N
    return A.astype(np.float32)


def small_int_matrix(m: int, n: int, seed: int, lim: int = 8) -> np.ndarray:
    return rng(seed).integers(-lim, lim + 1, size=(m, n)).astype(np.float32)


def spectrum_matrix_torch(s, seed: int, device="cuda"):
    """Same construction as spectrum_matrix(method='hadamard') with torch on `device` (FP64 math,
    FP32 result) for the large RSVD input (16384^2): A = P1 (H/sqrtN) D1 diag(s) D2 (H/sqrtN) P2^T."""
    import torch
    s = torch.as_tensor(np.asarray(s), dtype=torch.float64, device=device)
    N = s.shape[0]
    assert N & (N - 1) == 0
    g = rng(seed)
    d1 = torch.as_tensor(g.choice([-1.0, 1.0], N), device=device)
    d2 = torch.as_tensor(g.choice([-1.0, 1.0], N), device=device)
    p1 = torch.as_tensor(np.argsort(g.permutation(N)), device=device)
    p2 = torch.as_tensor(np.argsort(g.permutation(N)), device=device)

    def fwht_rows(X):
        n = X.shape[0]
        h = 1
        while h < n:
            Xv = X.view(n // (2 * h), 2, h, -1)
            a = Xv[:, 0].clone()
            b = Xv[:, 1]
            Xv[:, 0] = a + b
            Xv[:, 1] = a - b
            h *= 2
        return X

    M = torch.diag(s * d2)
    M = fwht_rows(M) / np.sqrt(N)
    M = M.t().contiguous()
    M = M[:, p2]
    M = d1[:, None] * M
    A = fwht_rows(M) / np.sqrt(N)
    A = A[p1]
    return A.to(torch.float32).contiguous()
