"""RandNLA harness on the GPU (SURVEY §2 A7 / A25, §8d "Pipelines").

Randomized SVD (Alg 1) and RP-HOSVD (Alg 2). The paper uses
SHGEMM for the random projection only (Alg 1 line 1; Alg 2 line 2) and cuBLAS/cuSOLVER for
everything else; so does this harness: the projection goes through the C ABI (`shgemm` /
`project`), QR/SVD/other products are torch.linalg / torch.matmul calls (cuSOLVER / cuBLAS FP32,
TF32 disabled). `projection="sgemm"` is the FP32 baseline of the paper's speedup figures (P:712:
"the random matrix is FP16 when using SHGEMM, otherwise FP32"): the same Gaussian stream kept in
FP32 (OMEGA_SPEC §6 values before FP16 rounding) and a cuBLAS SGEMM. Per-line device times are
recorded with CUDA events (the Fig 8 / Fig 9 breakdowns).

`gemm="tcec"` also moves the pipelines' other FP32 products onto the tensor cores
with the library's TCEC-SGEMM (Eqs 5-9): RSVD line 3 (B = Q^T A, computed as
B^T = A^T Q with A read in place) and the RP-HOSVD core contractions
(Alg 2 line 5). `gemm="sgemm"` keeps them on cuBLAS FP32 (TF32 off) as in the paper.
"""
from __future__ import annotations

import contextlib

import torch

from . import gen_omega, gen_omega_tiled, project, project_workspace_size, shgemm, synth, tcec_sgemm


@contextlib.contextmanager
def _fp32_matmul():
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        yield
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


class _Timer:
    def __init__(self, enabled=True):
        self.enabled = enabled
        self.marks = []

    def mark(self, name):
        if self.enabled:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.marks.append((name, e))

    def result(self):
        if not self.enabled or len(self.marks) < 2:
            return {}
        torch.cuda.synchronize()
        out = {}
        for (name, e0), (_, e1) in zip(self.marks[:-1], self.marks[1:]):
            out[name] = out.get(name, 0.0) + e0.elapsed_time(e1)
        out["total"] = self.marks[0][1].elapsed_time(self.marks[-1][1])
        return out


def _qr_pos(Y):
    Q, R = torch.linalg.qr(Y)
    d = torch.sign(torch.diagonal(R))
    d = torch.where(d == 0, torch.ones_like(d), d)
    return Q * d[None, :]


def cholqr2_async(Y: torch.Tensor):
    """(Q, bad) for Y = QR (R diagonal > 0, like _qr_pos) by CholeskyQR2 with FP64 Gram matrices:
    L1 = chol(Y^T Y), Q1 = Y L1^-T, then once more on Q1 (the second pass restores orthogonality to
    FP32 level for cond(Y) up to ~1e7). Tall-skinny QR as GEMMs + a tiny Cholesky + a tiny
    triangular inverse instead of cuSOLVER's panel factorization (16384 x 272: 1.2 vs 4.6 ms, DESIGN.md
    §8). Nothing synchronizes: `bad` is a device tensor, nonzero if a Gram matrix was not numerically
    positive definite (then Q is garbage and the caller recomputes with Householder)."""
    X = Y.double()
    n = X.shape[1]
    eye = torch.eye(n, dtype=torch.float64, device=Y.device)
    bad = torch.zeros((), dtype=torch.int32, device=Y.device)
    for _ in range(2):
        L, info = torch.linalg.cholesky_ex(X.t() @ X)
        bad = bad + info.to(torch.int32)
        X = X @ torch.linalg.solve_triangular(L, eye, upper=False).t()
    return X.to(Y.dtype), bad


def cholqr2(Y: torch.Tensor) -> torch.Tensor:
    """cholqr2_async with the Householder fallback applied (one synchronization)."""
    Q, bad = cholqr2_async(Y)
    return _qr_pos(Y) if int(bad) != 0 else Q


def gram_svd(Bt: torch.Tensor, p: int):
    """Top-p SVD of B = Bt^T (nhat x N, nhat small) from the FP64 eigendecomposition of B B^T:
    B B^T = U' diag(S^2) U'^T, V = B^T U' S^-1. Singular values carry a relative error
    ~ u64 (S_1 / S_i)^2, so the route is for the well-separated leading p of a randomized SVD;
    U S V^T = U' U'^T B exactly up to rounding, so the reconstruction is unaffected."""
    B64 = Bt.double()
    w, U = torch.linalg.eigh(B64.t() @ B64)
    w, U = w.flip(0)[:p], U.flip(1)[:, :p]
    S = torch.sqrt(torch.clamp(w, min=0.0))
    V = (B64 @ U) / torch.clamp(S, min=torch.finfo(torch.float64).tiny)[None, :]
    return U.float(), S.float(), V.float()


def omega_fp32(k: int, n: int, seed: int = 0, stream_id: int = 0, device="cuda") -> torch.Tensor:
    """FP32 Gaussian k x n (column-major view): the SAME counter-based draws as gen_omega's FP16 Omega
    (OMEGA_SPEC §2-3 addressing, §6 FP32 output) before the RN16 rounding, so the SGEMM baseline
    and SHGEMM project with the same random matrix up to its FP16 rounding."""
    return synth("gauss", seed, stream_id, n, k, device=device).t()


def rsvd(A: torch.Tensor, p: int, s: int = 10, seed: int = 0, dist="gaussian", projection="shgemm",
         timing: bool = False, gemm: str = "sgemm", factor: str = "cusolver", check: bool = True):
    """Alg 1: Y = A Omega; Q = QR(Y); B = Q^T A; (U', S, V) = tSVD(B, p); U = Q U'.
    factor='cusolver' (the paper's: Householder QR and SVD from cuSOLVER) or 'gram' (CholeskyQR2 and
    the FP64 Gram-eigh SVD; needs gemm='tcec' for B^T)."""
    if gemm not in ("sgemm", "tcec"):
        raise ValueError(gemm)
    if factor not in ("cusolver", "gram") or (factor == "gram" and gemm != "tcec"):
        raise ValueError(factor)
    m, n = A.shape
    nhat = p + s
    t = _Timer(timing)
    with _fp32_matmul():
        t.mark("1_projection")
        if projection == "shgemm":
            Om = gen_omega(n, nhat, seed=seed, dist=dist, device=A.device)
            Y = shgemm(A, Om)
        elif projection == "sgemm":
            Om = omega_fp32(n, nhat, seed=seed, device=A.device)
            Y = A @ Om
        else:
            raise ValueError(projection)
        t.mark("2_qr")
        bad = None
        if factor == "gram":
            Q, bad = cholqr2_async(Y)
        else:
            Q = _qr_pos(Y)
        t.mark("3_QtA")
        B = tcec_sgemm(A.t(), Q).t() if gemm == "tcec" else Q.t() @ A
        t.mark("4_svd")
        if factor == "gram":
            Uh, S, V = gram_svd(B.t(), p)
        else:
            Uh, S, Vt = torch.linalg.svd(B, full_matrices=False)
            V = Vt[:p].t()
        t.mark("5_QU")
        U = Q @ Uh[:, :p]     # 16384 x 272 x 256: launch-bound either way, left on cuBLAS
        t.mark("end")
    if check and bad is not None and int(bad) != 0:     # Gram not positive definite: redo with Householder QR
        return rsvd(A, p, s, seed, dist, projection, timing, gemm, "cusolver")
    # check=False (CUDA-graph capture: no synchronisation allowed): the caller checks "bad"
    return {"U": U, "S": S[:p], "V": V, "Q": Q, "times_ms": t.result(), "bad": bad}


def reconstruction_error(A, U, S, V) -> float:
    """||A - U diag(S) V^T||_F / ||A||_F, evaluated in FP64 on the device."""
    A64 = A.double()
    R = A64 - (U.double() * S.double()[None, :]) @ V.double().t()
    return float(torch.linalg.norm(R) / torch.linalg.norm(A64))


def unfold(T, mode):
    return torch.movedim(T, mode, 0).reshape(T.shape[mode], -1)


def mode_product(T, M, mode):
    """T x_mode M with M (I_mode x J): contracts M^T . unfold_mode(T) (reading R14)."""
    out = torch.tensordot(T, M, dims=([mode], [0]))
    return torch.movedim(out, -1, mode)


def core_tcec(T: torch.Tensor, Qs) -> torch.Tensor:
    """g = T x_1 Q_1^T ... x_N Q_N^T by TCEC-SGEMM: each step contracts the LEADING mode of the
    current C-order tensor, G'[rest, j] = sum_i g[i, rest] Q[i, j] — an MN-major A read in place
    (the (I x rest) view transposed) times an N-major Q — which moves the new mode to the end; after
    N steps the modes are back in order (J_1, ..., J_N)."""
    g = T.contiguous()
    for Q in Qs:
        I = g.shape[0]
        rest = g.shape[1:]
        g = tcec_sgemm(g.reshape(I, -1).t(), Q).reshape(*rest, Q.shape[1])
    return g


def _tc_view(dims, mode) -> bool:
    """True if project() reads the mode-`mode` unfolding of a 16-B-aligned C-order tensor with `dims`
    on the tcgen05 path (the only path that streams a caller's k-tiled Omega; csrc/api.cu
    project_impl): mode 0 is a K-major matrix with row stride K (K % 4 == 0), the last mode an M-major
    view with row stride M (M % 4 == 0), a middle mode a 3-D view (S % 32 == 0) or a padded copy."""
    M, K = dims[mode], 1
    for i, d in enumerate(dims):
        if i != mode:
            K *= d
    S = 1
    for d in dims[mode + 1:]:
        S *= d
    if mode == 0:
        return K % 4 == 0
    if S == 1:
        return M % 4 == 0
    return True


def rp_hosvd(T: torch.Tensor, ranks, seed: int = 0, dist="gaussian", projection="shgemm", timing=False,
             gemm: str = "sgemm", factor: str = "cusolver", check: bool = True, pregen: bool = True):
    """Alg 2: for each mode W = A'_(i) Omega_(i) (project, stream_id = mode), Q_i = QR(W);
    g = A x_1 Q_1^T ... x_N Q_N^T. factor='gram': CholeskyQR2 for the QRs. pregen=False: each
    project() generates its Omega_(i) itself (in-kernel by default) instead of the side stream."""
    if gemm not in ("sgemm", "tcec") or factor not in ("cusolver", "gram"):
        raise ValueError((gemm, factor))
    t = _Timer(timing)
    Qs, bads = [], []
    ws = None
    oms, ready = [None] * len(ranks), [None] * len(ranks)
    if projection == "shgemm":   # one persistent scratch buffer (Omega_(i) + split-K partials) for all modes
        nbytes = max(project_workspace_size(list(T.shape), i, J) for i, J in enumerate(ranks))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=T.device)
        if pregen and T.is_contiguous() and T.data_ptr() % 16 == 0:
            # every Omega_(i) generated up front on a side stream (k-tiled, as project() streams it):
            # the generator (ALU-bound) fills the gaps of the latency-bound QRs between projections
            side = torch.cuda.Stream(device=T.device)
            side.wait_stream(torch.cuda.current_stream())
            numel = T.numel()
            with torch.cuda.stream(side):
                for i, J in enumerate(ranks):
                    if not _tc_view(list(T.shape), i):   # project() generates its own Omega there
                        continue
                    oms[i] = gen_omega_tiled(numel // T.shape[i], J, seed=seed, dist=dist, stream_id=i,
                                             device=T.device)
                    ready[i] = torch.cuda.Event()
                    ready[i].record(side)
    with _fp32_matmul():
        for i, J in enumerate(ranks):
            t.mark("2_projection")
            if projection == "shgemm" and oms[i] is not None:
                torch.cuda.current_stream().wait_event(ready[i])
                oms[i].record_stream(torch.cuda.current_stream())
                W = project(T, i, J, workspace=ws, omega=oms[i])
            elif projection == "shgemm":
                W = project(T, i, J, seed=seed, dist=dist, workspace=ws)
            elif projection == "sgemm":
                Ui = unfold(T, i)
                Om = omega_fp32(Ui.shape[1], J, seed=seed, stream_id=i, device=T.device)
                W = Ui @ Om
            else:
                raise ValueError(projection)
            t.mark("3_qr")
            if factor == "gram":
                Q, b = cholqr2_async(W)
                bads.append(b)
                Qs.append(Q)
            else:
                Qs.append(_qr_pos(W))
        t.mark("5_core")
        if gemm == "tcec":
            g = core_tcec(T, Qs)
        else:
            g = T
            for i, Q in enumerate(Qs):
                g = mode_product(g, Q, i)
        t.mark("end")
    if check and bads and int(sum(bads)) != 0:
        return rp_hosvd(T, ranks, seed, dist, projection, timing, gemm, "cusolver", pregen=pregen)
    # check=False (CUDA-graph capture: no synchronisation allowed): the caller checks "bad"
    return {"core": g, "Q": Qs, "times_ms": t.result(), "bad": sum(bads) if bads else None}


def hosvd_error(T, core, Qs) -> float:
    """||A - g x_1 Q_1 ... x_N Q_N||_F / ||A||_F in FP64."""
    R = core.double()
    for i, Q in enumerate(Qs):
        R = mode_product(R, Q.double().t(), i)
    T64 = T.double()
    return float(torch.linalg.norm(T64 - R) / torch.linalg.norm(T64))
