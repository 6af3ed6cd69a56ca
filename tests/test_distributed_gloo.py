"""Multi-process (gloo, CPU) tests of the communication-avoiding distributed pipelines of
paper_2304_04612_b200/distributed.py: TSQR + all-reduce(B^T) RSVD on a
row-sharded A, and K-sharded RP-HOSVD on mode-0 slabs (all-gather W_0, all-reduce W_i, all-reduce
core). The exchange logic is the product's; the LOCAL arithmetic here is the CPU oracle's (test
infrastructure: projections = oracle.gemm_y32 with the oracle's Omega rows at the slab's offset),
so every rank's pieces are pinned independently of the CUDA path. Bars: the sharded pipelines
reproduce the single-process FP32 oracle pipelines' residuals within 1e-4 relative (reading R10)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleOps:
    """CPU stand-ins for the device steps, built from the oracle (tests only)."""

    def project_rows(self, A_local, n, seed, dist_kind):
        import oracle
        A = A_local.numpy()
        om = oracle.omega_f16(A.shape[1], n, seed=seed, dist=dist_kind)
        return torch.from_numpy(oracle.gemm_y32(A, om))

    def project_slab(self, T_local, mode, n, seed, dist_kind, omega_row0, k_total):
        import oracle
        from oracle import pipelines as opl
        Ai = np.ascontiguousarray(opl.unfold(T_local.numpy(), mode))
        om = oracle.omega_f16(Ai.shape[1], n, seed=seed, dist=dist_kind, stream_id=mode, row0=omega_row0,
                              k_total=k_total)
        return torch.from_numpy(oracle.gemm_y32(Ai, om))

    def gemm_tn(self, X, Q):
        return X.t() @ Q

    def contract_leading(self, g, Q):
        return torch.tensordot(g, Q, dims=([0], [0]))

    def matmul(self, X, Y):
        return X @ Y

    def qr(self, Y):
        return torch.linalg.qr(Y)

    def svd(self, B):
        return torch.linalg.svd(B, full_matrices=False)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, job, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2304_04612_b200 import distributed as D
        from paper_2304_04612_b200.shard import row_partition
        ops = OracleOps()
        if job["kind"] == "rsvd":
            m, n, p, s = job["m"], job["n"], job["p"], job["s"]
            if job.get("exact_rank"):
                rng = np.random.default_rng(0)
                A = (rng.standard_normal((m, p)) @ rng.standard_normal((p, n))).astype(np.float32)
            else:
                A = synth.spectrum_matrix(synth.spectrum("exp", max(m, n), p, 1e-2), seed=3)[:m, :n]
                A = np.ascontiguousarray(A, dtype=np.float32)
            r0, rows = row_partition(m, world, rank)
            out = D.dist_rsvd(torch.from_numpy(A[r0:r0 + rows]), p, s, seed=4, ops=ops)
            U = D.all_gather_rows(out["U"], [row_partition(m, world, r)[1] for r in range(world)])
            Q = D.all_gather_rows(out["Q"], [row_partition(m, world, r)[1] for r in range(world)])
            if rank == 0:
                q.put({"A": A, "U": U.numpy(), "S": out["S"].numpy(), "V": out["V"].numpy(), "Q": Q.numpy(),
                       "exch": out["exchange_bytes"]})
        else:
            dims, ranks = job["dims"], job["ranks"]
            T = synth.alg3_tensor(dims, ranks, pad=2, seed=5, noise=1e-2)
            s0, nl = D.slab_partition(dims[0], world, rank)
            out = D.dist_rp_hosvd(torch.from_numpy(np.ascontiguousarray(T[s0:s0 + nl])), dims, ranks, seed=2,
                                  ops=ops)
            if rank == 0:
                q.put({"T": T, "core": out["core"].numpy(), "Q": [Q.numpy() for Q in out["Q"]]})
    finally:
        dist.destroy_process_group()


def _run(world, job):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, job, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3, 4])
def test_dist_rsvd_matches_oracle_pipeline(orc, world):
    from oracle import pipelines as opl
    m, n, p, s = 301, 200, 12, 6
    res = _run(world, {"kind": "rsvd", "m": m, "n": n, "p": p, "s": s})
    A = res["A"]
    e_dist = opl.reconstruction_error(A, res["U"], res["S"], res["V"])
    e_or = opl.rsvd(A, p, s, seed=4, precision="f32")["residual"]
    assert e_dist > 1e-3
    assert abs(e_dist - e_or) <= 1e-4 * e_or, (e_dist, e_or)
    Q = res["Q"].astype(np.float64)
    assert np.abs(Q.T @ Q - np.eye(p + s)).max() < 1e-5          # TSQR's Q is orthonormal
    assert res["exch"]["qta_allreduce"] == n * (p + s) * 4         # B^T all-reduce: N x nhat, not m x n


def test_dist_rsvd_short_shards_exact_rank(orc):
    """Shards shorter than nhat (m_g = 11 < 16): the reduced local QR / padded R path; an exact
    rank-p matrix is recovered to FP32 level."""
    from oracle import pipelines as opl
    res = _run(2, {"kind": "rsvd", "m": 22, "n": 40, "p": 6, "s": 10, "exact_rank": True})
    assert opl.reconstruction_error(res["A"], res["U"], res["S"], res["V"]) <= 1e-5


@pytest.mark.parametrize("world,dims,ranks", [(2, (24, 20, 18), (6, 6, 6)), (3, (4, 20, 18), (4, 6, 6)),
                                              (3, (25, 16, 12), (6, 6, 6))])
def test_dist_rp_hosvd_matches_oracle_pipeline(orc, world, dims, ranks):
    """K-sharded unfoldings (omega_row0 = s0 * S_i) + all-reduce; world 3 with I0 = 4 has an
    empty slab on the last rank."""
    from oracle import pipelines as opl
    res = _run(world, {"kind": "hosvd", "dims": dims, "ranks": ranks})
    T = res["T"]
    e_dist = opl.hosvd_error(T, res["core"], res["Q"])
    e_or = opl.rp_hosvd(T, ranks, seed=2, precision="f32")["residual"]
    assert abs(e_dist - e_or) <= 1e-4 * e_or, (e_dist, e_or)


def test_slab_omega_rows_are_the_global_unfolding_columns(orc):
    """The addressing K-sharding relies on: a mode-0 slab's mode-i unfolding is the column block
    [s0 * S_i, (s0 + n) * S_i) of the full unfolding, and Omega rows generated at that offset equal
    the full Omega's rows there (counter-based generator, OMEGA_SPEC §2)."""
    from oracle import pipelines as opl
    from paper_2304_04612_b200.distributed import slab_partition
    T = np.arange(5 * 4 * 3, dtype=np.float32).reshape(5, 4, 3)
    for mode in (1, 2):
        full = opl.unfold(T, mode)
        S_i = full.shape[1] // T.shape[0]
        om_full = orc.omega_f16(full.shape[1], 7, seed=9, stream_id=mode)
        for rank in range(2):
            s0, nl = slab_partition(5, 2, rank)
            part = opl.unfold(T[s0:s0 + nl], mode)
            np.testing.assert_array_equal(part, full[:, s0 * S_i:(s0 + nl) * S_i])
            om = orc.omega_f16(part.shape[1], 7, seed=9, stream_id=mode, row0=s0 * S_i, k_total=full.shape[1])
            np.testing.assert_array_equal(om, om_full[s0 * S_i:(s0 + nl) * S_i])
