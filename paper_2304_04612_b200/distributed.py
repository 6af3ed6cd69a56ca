"""Communication-avoiding distributed RandNLA (SURVEY §8e "downstream" and §8f NEXT-3).

The hot path (the random projection) shards with NO collective: every rank regenerates the same
Omega from the shared seed (OMEGA_SPEC §2) and projects its own rows (shard.py, bench.py). What
follows the projection in the paper's pipelines does need data from every rank; this module keeps
that exchange at the size of the small factors instead of gathering Y or A:

Randomized SVD, Alg 1, A row-sharded (rank g owns rows [r0_g, r0_g + m_g)):
  line 1  Y_g = A_g . Omega                                     local (SHGEMM), no communication
  line 2  TSQR: Y_g = Q_g R_g locally; ALL-GATHER the G small R_g (nhat x nhat); QR of the stacked
          R's = Q_s R; Q = blockdiag(Q_g) . Q_s, i.e. rank g keeps Q_g . Q_s[g]   (R diag >= 0)
  line 3  B^T = sum_g A_g^T Q_g: local TCEC-SGEMM (B^T = A^T Q, A read in place) + one ALL-REDUCE
          of N x nhat (4 MiB for cfg4, 17 MiB for cfg2) — instead of the 4 GiB all-gather of Y
  line 4  SVD of B, replicated on every rank (nhat x N)
  line 5  U_g = Q_g U'[:, :p]                                   local rows of U

RP-HOSVD, Alg 2, the tensor sharded in slabs along mode 0 (rank g owns
i_0 in [s0_g, s0_g + n_g)):
  line 2  mode 0: the slab's rows of W_0 are complete (its unfolding columns are all local):
          ALL-GATHER the row blocks (I_0 x J_0 FP32, 256 KiB for cfg3).
          mode i >= 1: the slab holds a contiguous range of the unfolding's COLUMNS
          ([s0_g * S_i, (s0_g + n_g) * S_i), S_i = prod_{l != 0, i} I_l), so W_i = sum_g of the
          slab products with the matching rows of Omega_(i) (C ABI `project_shard`, omega_row0):
          one ALL-REDUCE of I_i x J_i per mode — K-sharding.
  line 3  QR of each W_i, replicated.
  line 5  core: g = sum_g T_g x_0 Q_0[slab_g]^T x_1 Q_1^T ... : local TCEC-SGEMM contractions and one
          ALL-REDUCE of J_0 x ... x J_{N-1} (1 MiB for cfg3).

The local compute goes through `ops` (default: the library's kernels on the rank's GPU plus
torch.linalg for the small dense factorizations). Collectives are torch.distributed over NCCL on
GPUs; with the gloo backend (CPU tests) CUDA tensors are staged through host memory.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class DeviceOps:
    """The product's local steps: SHGEMM projections and TCEC-SGEMM products from libshgemm.so,
    QR / SVD from torch.linalg (cuSOLVER) in FP32."""

    def project_rows(self, A_local: torch.Tensor, n: int, seed: int, dist_kind: str) -> torch.Tensor:
        from . import gen_omega, shgemm
        Om = gen_omega(A_local.shape[1], n, seed=seed, dist=dist_kind, device=A_local.device)
        return shgemm(A_local, Om)

    def project_slab(self, T_local: torch.Tensor, mode: int, n: int, seed: int, dist_kind: str, omega_row0: int,
                     k_total: int) -> torch.Tensor:
        from . import project
        return project(T_local, mode, n, seed=seed, dist=dist_kind, omega_row0=omega_row0, k_total=k_total)

    def gemm_tn(self, X: torch.Tensor, Q: torch.Tensor) -> torch.Tensor:
        """X^T Q (X read in place as an MN-major operand)."""
        from . import tcec_sgemm
        return tcec_sgemm(X.t(), Q)

    def contract_leading(self, g: torch.Tensor, Q: torch.Tensor) -> torch.Tensor:
        """G'[rest, j] = sum_i g[i, rest] Q[i, j] (the new mode moves to the end)."""
        from . import tcec_sgemm
        I = g.shape[0]
        return tcec_sgemm(g.reshape(I, -1).t(), Q).reshape(*g.shape[1:], Q.shape[1])

    def matmul(self, X: torch.Tensor, Y: torch.Tensor) -> torch.Tensor:
        return X @ Y

    def qr(self, Y: torch.Tensor):
        return torch.linalg.qr(Y)

    def svd(self, B: torch.Tensor):
        return torch.linalg.svd(B, full_matrices=False)


# ------------------------------------------------------------------------------------ collectives
def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _staged(t: torch.Tensor, group):
    """gloo has no CUDA collectives for every op: stage CUDA tensors through host memory."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        return t.cpu(), True
    return t, False


def all_reduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    world, _ = _world(group)
    if world == 1:
        return t
    x, staged = _staged(t.contiguous(), group)
    dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)
    return x.to(t.device) if staged else x


def all_gather_rows(t: torch.Tensor, rows_per_rank, group=None) -> torch.Tensor:
    """Concatenate every rank's (rows_g x n) block in rank order (blocks padded to the max)."""
    world, rank = _world(group)
    if world == 1:
        return t
    per = max(rows_per_rank)
    pad = torch.zeros((per,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    x, staged = _staged(pad, group)
    parts = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(parts, x, group=group)
    out = torch.cat([p[:r] for p, r in zip(parts, rows_per_rank)], 0)
    return out.to(t.device) if staged else out


def _sign_fix(Q, R):
    d = torch.sign(torch.diagonal(R))
    d = torch.where(d == 0, torch.ones_like(d), d)
    return Q * d[None, :], R * d[:, None]


# ------------------------------------------------------------------------------------ TSQR
def tsqr(Y_local: torch.Tensor, group=None, ops=None):
    """Q_local (this rank's rows of Q) and the replicated R of Y = Q R for a row-sharded tall Y,
    R with a non-negative diagonal. One all-gather of the G (n x n) R factors."""
    ops = ops or DeviceOps()
    n = Y_local.shape[1]
    world, rank = _world(group)
    Qg, Rg = ops.qr(Y_local)                      # reduced: Qg m_g x r_g, Rg r_g x n, r_g = min(m_g, n)
    r = Rg.shape[0]
    if world == 1:
        return _sign_fix(Qg, Rg)
    Rpad = torch.zeros((n, n), dtype=Rg.dtype, device=Rg.device)
    Rpad[:r] = Rg
    Rs = all_gather_rows(Rpad, [n] * world, group)            # (G n) x n, identical on every rank
    Qs, R = ops.qr(Rs)
    Qs, R = _sign_fix(Qs, R)
    Q_local = ops.matmul(Qg, Qs[rank * n: rank * n + r].contiguous())
    return Q_local, R


# ------------------------------------------------------------------------------------ RSVD
def dist_rsvd(A_local: torch.Tensor, p: int, s: int = 10, seed: int = 0, dist_kind: str = "gaussian",
              group=None, ops=None):
    """Alg 1 on a row-sharded A (this rank's rows A_local). Returns this rank's rows of U, the
    replicated S and V, and the per-step exchange sizes (bytes) for the record."""
    ops = ops or DeviceOps()
    nhat = p + s
    Y = ops.project_rows(A_local, nhat, seed, dist_kind)                  # line 1: no communication
    Q_local, _ = tsqr(Y, group, ops)                                      # line 2: all-gather of R's
    Bt = all_reduce_sum(ops.gemm_tn(A_local, Q_local), group)             # line 3: one all-reduce
    Uh, S, Vt = ops.svd(Bt.t())                                           # line 4: replicated
    U_local = ops.matmul(Q_local, Uh[:, :p].contiguous())                 # line 5: local
    world, _ = _world(group)
    exch = {"tsqr_allgather": world * nhat * nhat * 4, "qta_allreduce": Bt.numel() * 4}
    return {"U": U_local, "S": S[:p], "V": Vt[:p].t(), "Q": Q_local, "exchange_bytes": exch}


# ------------------------------------------------------------------------------------ RP-HOSVD
def slab_partition(I0: int, world: int, rank: int):
    """(s0, n) of rank `rank`'s slab along mode 0: contiguous blocks of ceil(I0 / world)."""
    per = (I0 + world - 1) // world
    s0 = min(I0, rank * per)
    return s0, max(0, min(I0, s0 + per) - s0)


def dist_rp_hosvd(T_local: torch.Tensor, dims, ranks, seed: int = 0, dist_kind: str = "gaussian", group=None,
                  ops=None):
    """Alg 2 on a tensor sharded in mode-0 slabs: T_local = T[s0 : s0 + n] of the full `dims`.
    Returns the replicated core and factor matrices Q_i."""
    ops = ops or DeviceOps()
    dims = [int(d) for d in dims]
    N = len(dims)
    world, rank = _world(group)
    s0, nloc = slab_partition(dims[0], world, rank)
    if tuple(T_local.shape) != (nloc, *dims[1:]):
        raise ValueError(f"slab shape {tuple(T_local.shape)} != {(nloc, *dims[1:])}")
    Qs = []
    for i, J in enumerate(ranks):
        K = 1
        for l, d in enumerate(dims):
            if l != i:
                K *= d
        if i == 0:
            W0 = (ops.project_slab(T_local, 0, J, seed, dist_kind, 0, K) if nloc else
                  torch.zeros((0, J), dtype=torch.float32, device=T_local.device))
            W = all_gather_rows(W0, [slab_partition(dims[0], world, r)[1] for r in range(world)], group)
        else:
            S_i = K // dims[0]
            if nloc:
                Wp = ops.project_slab(T_local, i, J, seed, dist_kind, s0 * S_i, K)
            else:
                Wp = torch.zeros((dims[i], J), dtype=torch.float32, device=T_local.device)
            W = all_reduce_sum(Wp, group)
        Q, R = ops.qr(W)
        Qs.append(_sign_fix(Q, R)[0])
    if nloc:
        g = ops.contract_leading(T_local.contiguous(), Qs[0][s0:s0 + nloc].contiguous())
        for Q in Qs[1:]:
            g = ops.contract_leading(g, Q)
    else:
        g = torch.zeros(tuple(Q.shape[1] for Q in Qs), dtype=torch.float32, device=T_local.device)
    core = all_reduce_sum(g.contiguous(), group)
    return {"core": core, "Q": Qs}
