"""GPU tests of the distributed pipelines' device path (NEXT-3, paper_2304_04612_b200/distributed.py):
`project_shard` (K-sharded unfoldings: a slab's projection with the full Omega's rows at its column
offset) against the oracle, and TSQR/all-reduce RSVD and K-sharded RP-HOSVD with the library's
kernels (DeviceOps) — in one process and as two gloo ranks sharing cuda:0 — against the FP32
oracle pipelines (reading R10: residuals within 1e-4 relative)."""
import os
import socket

import numpy as np
import pytest

import synth
from gpu_common import check_bars, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def shg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_04612_b200 import _build
    _build.build()
    import paper_2304_04612_b200 as m
    return m


@pytest.mark.parametrize("dims", [(40, 96, 72), (9, 128, 64), (12, 33, 17)])
def test_project_shard_slabs(shg, orc, dims):
    """Each mode-0 slab's W_i uses Omega_(i) rows [s0 * S_i, ...) (bit-exact generator) and meets
    the bars; the slab sum equals the full projection to FP32 rounding."""
    from oracle import pipelines as opl
    from paper_2304_04612_b200.distributed import slab_partition
    T = synth.gaussian(int(np.prod(dims)), 1, seed=3).reshape(dims)
    Tc = torch.from_numpy(T).cuda()
    for mode in range(3):
        K = int(np.prod(dims)) // dims[mode]
        W_full = shg.project(Tc, mode, 24, seed=1)
        acc = torch.zeros_like(W_full, dtype=torch.float64)
        for rank in range(2):
            s0, nl = slab_partition(dims[0], 2, rank)
            slab = np.ascontiguousarray(T[s0:s0 + nl])
            row0 = 0 if mode == 0 else s0 * (K // dims[0])
            W = shg.project(torch.from_numpy(slab).cuda(), mode, 24, seed=1, omega_row0=row0, k_total=K)
            torch.cuda.synchronize()
            Ai = np.ascontiguousarray(opl.unfold(slab, mode))
            om = orc.omega_f16(Ai.shape[1], 24, seed=1, stream_id=mode, row0=row0, k_total=K)
            check_bars(orc, Ai, om, to_np(W))
            if mode == 0:
                acc[s0:s0 + nl] += W.double()
            else:
                acc += W.double()
        rel = float(torch.linalg.norm(acc - W_full.double()) / torch.linalg.norm(W_full.double()))
        assert rel < 2e-6, (mode, rel)


def test_project_shard_rejects_bad_offsets(shg):
    T = torch.randn(4, 8, 8, device="cuda")
    with pytest.raises(shg.SHGError):
        shg.project(T, 1, 8, omega_row0=-1)
    with pytest.raises(shg.SHGError):
        shg.project(T, 1, 8, omega_row0=10, k_total=20)     # 10 + 32 > 20


def test_dist_rsvd_single_rank_device(shg, orc):
    from oracle import pipelines as opl
    from paper_2304_04612_b200 import distributed as D
    A = synth.spectrum_matrix(synth.spectrum("exp", 512, 22, 1e-2), seed=3)
    out = D.dist_rsvd(torch.from_numpy(A).cuda(), 22, 10, seed=4)
    e = opl.reconstruction_error(A, to_np(out["U"]), to_np(out["S"]), to_np(out["V"]))
    e_or = opl.rsvd(A, 22, 10, seed=4, precision="f32")["residual"]
    assert abs(e - e_or) <= 1e-4 * e_or, (e, e_or)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2304_04612_b200 import distributed as D
        from paper_2304_04612_b200.shard import row_partition
        m = 1000
        A = synth.spectrum_matrix(synth.spectrum("exp", m, 22, 1e-2), seed=3)
        r0, rows = row_partition(m, world, rank)
        out = D.dist_rsvd(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda(), 22, 10, seed=4)
        U = D.all_gather_rows(out["U"], [row_partition(m, world, r)[1] for r in range(world)])
        dims, ranks = (48, 40, 36), (8, 8, 8)
        T = synth.alg3_tensor(dims, ranks, pad=2, seed=5, noise=1e-2)
        s0, nl = D.slab_partition(dims[0], world, rank)
        h = D.dist_rp_hosvd(torch.from_numpy(np.ascontiguousarray(T[s0:s0 + nl])).cuda(), dims, ranks, seed=2)
        if rank == 0:
            q.put({"A": A, "U": to_np(U), "S": to_np(out["S"]), "V": to_np(out["V"]), "T": T,
                   "core": to_np(h["core"]), "Q": [to_np(Q) for Q in h["Q"]]})
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_gloo(shg, orc):
    """world_size 2 (gloo, both ranks on cuda:0): the product's device path end to end."""
    import torch.multiprocessing as mp
    from oracle import pipelines as opl
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    e = opl.reconstruction_error(res["A"], res["U"], res["S"], res["V"])
    e_or = opl.rsvd(res["A"], 22, 10, seed=4, precision="f32")["residual"]
    assert abs(e - e_or) <= 1e-4 * e_or, (e, e_or)
    eh = opl.hosvd_error(res["T"], res["core"], res["Q"])
    eh_or = opl.rp_hosvd(res["T"], (8, 8, 8), seed=2, precision="f32")["residual"]
    assert abs(eh - eh_or) <= 1e-4 * eh_or, (eh, eh_or)
