"""Row-sharded multi-GPU SHGEMM projection (SURVEY §8e, a9 of §8a).

Rows of A are independent units: rank g of G owns rows [g*ceil(m/G), min(m, (g+1)*ceil(m/G))) of
A and of Y = A . Omega. Every rank regenerates the identical Omega from the shared seed with the
counter-based generator (OMEGA_SPEC.md §2: the value of Omega[i][j] depends only on (seed, stream,
i, j)), so there is NO collective on the data path. torch.distributed is used only for plumbing:
a barrier, the max-over-ranks timing, and (outside the hot path) an optional all-gather of Y; the
downstream pipelines use distributed.py instead (TSQR + all-reduce, no gather of Y).
"""
from __future__ import annotations

import zlib


def row_partition(m: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, rows) of rank `rank`: contiguous blocks of ceil(m / world) rows, the last possibly
    shorter or empty."""
    if world < 1 or not 0 <= rank < world or m < 0:
        raise ValueError("bad partition arguments")
    per = (m + world - 1) // world
    row0 = min(m, rank * per)
    return row0, max(0, min(m, row0 + per) - row0)


def checksum_bits(buf) -> int:
    """CRC32 of a tensor's / array's raw bytes (used to assert identical Omega on every rank)."""
    import numpy as np
    if hasattr(buf, "detach"):
        buf = buf.detach().cpu().contiguous().numpy()
    return zlib.crc32(np.ascontiguousarray(buf).view(np.uint8).tobytes())


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank float over the process group (timing rule: the slowest rank counts)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    backend = dist.get_backend(group)
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def project_rows(A_local, k: int, n: int, seed: int = 0, dist: str = "gaussian", out=None):
    """This rank's Y block: Omega regenerated locally (same seed on every rank) and multiplied with
    the rank's row block of A through the C ABI. Returns (Y_local, Omega)."""
    import paper_2304_04612_b200 as shg
    Om = shg.gen_omega(k, n, seed=seed, dist=dist, device=A_local.device)
    Y = shg.shgemm(A_local, Om, out=out)
    return Y, Om


def gather_rows(Y_local, m: int, group=None):
    """Downstream only (not the hot path): all-gather the row blocks into the full m x n Y."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = (m + world - 1) // world
    n = Y_local.shape[1]
    pad = torch.zeros((per, n), dtype=Y_local.dtype, device=Y_local.device)
    pad[: Y_local.shape[0]] = Y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat(parts, 0)[:m]
