"""Pins for the oracle RandNLA pipelines (Alg 1; Alg 2)
and for the synthetic inputs they run on.

Pins: Eckart-Young (Theorem 1) closed forms vs direct tail sums; prescribed spectra
recovered by LAPACK SVD; the Halko expectation bound Eq 4 averaged over 100 seeds;
exact recovery of exact-rank inputs; naive index loops for unfold / mode product."""
import math

import numpy as np
import pytest

import synth
from oracle import pipelines as pl


@pytest.mark.parametrize("kind", ["linear", "exp"])
@pytest.mark.parametrize("s_p", [1e-1, 1e-2, 1e-3])
def test_eckart_young_closed_forms(kind, s_p):
    """P:684-691 closed forms == sqrt(sum_{i>=p} s_i^2) (readings c4-14, c4-15)."""
    N, p = 4096, 256
    s = synth.spectrum(kind, N, p, s_p)
    direct = math.sqrt(float(np.sum(s[p:] ** 2)))
    assert synth.eckart_young_floor(kind, N, p, s_p) == pytest.approx(direct, rel=1e-9)
    assert s[0] == 1.0 and (s[p] == pytest.approx(s_p))


@pytest.mark.parametrize("method", ["haar", "hadamard"])
def test_spectrum_matrix_has_prescribed_singular_values(method):
    s = synth.spectrum("exp", 256, 22, 1e-2)
    A = synth.spectrum_matrix(s, seed=3, method=method)
    sv = np.linalg.svd(A.astype(np.float64), compute_uv=False)
    assert np.allclose(sv, s, rtol=0, atol=2e-6)


def test_rsvd_exact_rank_recovery():
    rng = np.random.default_rng(0)
    A = (rng.standard_normal((300, 20)) @ rng.standard_normal((20, 400))).astype(np.float32)
    r32 = pl.rsvd(A, p=20, s=10, seed=1, precision="f32")
    r64 = pl.rsvd(A, p=20, s=10, seed=1, precision="f64")
    assert r32["residual"] < 1e-5 and r64["residual"] < 1e-6
    for r in (r32, r64):
        Q = r["U"].astype(np.float64)
        assert np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])) < 1e-4
        assert np.all(np.diff(r["S"]) <= 0)


@pytest.mark.parametrize("kind", ["linear", "exp"])
def test_rsvd_never_beats_eckart_young(kind):
    N, p, s_p = 512, 22, 1e-2
    s = synth.spectrum(kind, N, p, s_p)
    A = synth.spectrum_matrix(s, seed=5)
    floor = synth.eckart_young_floor(kind, N, p, s_p) / float(np.linalg.norm(A.astype(np.float64)))
    for seed in range(3):
        r = pl.rsvd(A, p=p, s=10, seed=seed, precision="f64")
        assert r["residual"] >= floor * (1 - 1e-6)
        assert r["residual"] < 3 * floor
        r32 = pl.rsvd(A, p=p, s=10, seed=seed, precision="f32")
        assert abs(r32["residual"] - r["residual"]) <= 1e-4 * r["residual"] + 2e-6


@pytest.mark.parametrize("kind,s_p", [("linear", 1e-3), ("exp", 1e-1)])
def test_halko_expectation_bound(kind, s_p, orc):
    """E||A - Q Q^T A||_F <= sqrt(1 + p/(s-1)) ||Sigma_2||_F (Eq 4), FP16 Omega
    (Theorems 2-5 justify the low-precision Gaussian). Mean over 100 seeds with 1.1 slack
    (reading c4-16)."""
    N, p, s = 512, 22, 10
    sig = synth.spectrum(kind, N, p, s_p)
    A = synth.spectrum_matrix(sig, seed=7)
    bound = pl.halko_bound(sig, p, s)
    errs = []
    for seed in range(100):
        om = orc.omega_f16(N, p + s, seed=seed)
        Y = orc.gemm_y64(A, om)
        Q, _ = np.linalg.qr(Y)
        errs.append(pl.projection_error(A, Q))
    assert np.mean(errs) <= 1.1 * bound
    assert min(errs) >= math.sqrt(float(np.sum(sig[p + s:] ** 2))) * (1 - 1e-6)


def test_unfold_matches_index_loops():
    dims = (2, 3, 4, 5)
    T = np.arange(np.prod(dims), dtype=np.float64).reshape(dims)
    for mode in range(4):
        U = pl.unfold(T, mode)
        rest = [d for i, d in enumerate(dims) if i != mode]
        assert U.shape == (dims[mode], int(np.prod(rest)))
        for idx in np.ndindex(*dims):
            others = [idx[i] for i in range(4) if i != mode]
            c = 0
            for o, d in zip(others, rest):
                c = c * d + o
            assert U[idx[mode], c] == T[idx]


def test_mode_product_matches_index_loops():
    rng = np.random.default_rng(1)
    dims = (3, 4, 2)
    T = rng.integers(-3, 4, size=dims).astype(np.float64)
    for mode in range(3):
        M = rng.integers(-3, 4, size=(dims[mode], 5)).astype(np.float64)
        G = pl.mode_product(T, M, mode)
        shp = list(dims)
        shp[mode] = 5
        assert G.shape == tuple(shp)
        for idx in np.ndindex(*shp):
            acc = 0.0
            for t in range(dims[mode]):
                src = list(idx)
                src[mode] = t
                acc += T[tuple(src)] * M[t, idx[mode]]
            assert G[idx] == acc
    # distinct modes commute (integer tensors, exact)
    M0 = rng.integers(-2, 3, size=(3, 2)).astype(np.float64)
    M2 = rng.integers(-2, 3, size=(2, 3)).astype(np.float64)
    a = pl.mode_product(pl.mode_product(T, M0, 0), M2, 2)
    b = pl.mode_product(pl.mode_product(T, M2, 2), M0, 0)
    assert np.array_equal(a, b)


def test_rp_hosvd_exact_multilinear_rank():
    """Alg 3 tensor of multilinear rank J - p is recovered exactly by Alg 2 with rank J."""
    T = synth.alg3_tensor((40, 36, 32), (12, 12, 12), pad=4, seed=3)
    r = pl.rp_hosvd(T, (12, 12, 12), seed=0, precision="f32")
    assert r["residual"] < 1e-5
    for Q in r["Q"]:
        Q = Q.astype(np.float64)
        assert np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])) < 1e-4
    assert r["core"].shape == (12, 12, 12)


def test_rp_hosvd_noisy_f32_vs_f64():
    T = synth.alg3_tensor((40, 36, 32), (12, 12, 12), pad=4, seed=4, noise=1e-2)
    r32 = pl.rp_hosvd(T, (12, 12, 12), seed=1, precision="f32")
    r64 = pl.rp_hosvd(T, (12, 12, 12), seed=1, precision="f64")
    assert r64["residual"] > 1e-3
    assert abs(r32["residual"] - r64["residual"]) <= 1e-4 * r64["residual"]


def test_alg3_tensor_rank():
    T = synth.alg3_tensor((30, 28, 26), (10, 10, 10), pad=3, seed=9)
    for mode in range(3):
        sv = np.linalg.svd(pl.unfold(T.astype(np.float64), mode), compute_uv=False)
        assert sv[6] > 1e-3 * sv[0] and sv[7] < 1e-5 * sv[0]


def test_cauchy_like_exceeds_fp16_range():
    A = synth.cauchy_like(256, seed=0)
    assert np.max(np.abs(A)) > 65504 and np.all(np.isfinite(A))
