"""Multi-process (world_size 2, gloo, CPU) tests of the row-sharded driver's host logic (§8e):
the row partition covers every row exactly once, every rank's regenerated Omega is identical
(checksums all-gathered), row blocks of the projection concatenate to the unsharded result, and the
timing reduction takes the max over ranks. The projection arithmetic on CPU here is the oracle's
(test infrastructure); the GPU path uses the same partition through bench.py / shard.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_04612_b200.shard import checksum_bits, max_over_ranks, row_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, k, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        row0, rows = row_partition(m, world, rank)
        A = synth.gaussian(m, k, seed=11)               # every rank can build the (small) test input
        om = oracle.omega_f16(k, n, seed=5)             # regenerated locally, same seed
        crc = torch.tensor([checksum_bits(om)], dtype=torch.int64)
        crcs = [torch.zeros_like(crc) for _ in range(world)]
        dist.all_gather(crcs, crc)
        Y_local = oracle.gemm_y32(A[row0:row0 + rows], om)
        per = (m + world - 1) // world
        pad = torch.zeros((per, n), dtype=torch.float32)
        pad[:rows] = torch.from_numpy(Y_local)
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        Y = torch.cat(parts, 0)[:m].numpy()
        t = max_over_ranks(float(rank + 1) * 1.5)
        if rank == 0:
            full = oracle.gemm_y32(A, om)
            q.put({"crcs": [int(c.item()) for c in crcs], "equal": bool(np.array_equal(Y, full)),
                   "tmax": t, "rows": [row_partition(m, world, r) for r in range(world)]})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [257, 128])
def test_two_rank_row_sharding_gloo(m):
    world, k, n = 2, 96, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, k, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(set(res["crcs"])) == 1          # identical Omega on every rank, no communication
    assert res["equal"]                        # concatenated shards == unsharded projection, bitwise
    assert res["tmax"] == 3.0                  # max over ranks
    covered = sorted(r for r0, c in res["rows"] for r in range(r0, r0 + c))
    assert covered == list(range(m))


@pytest.mark.parametrize("m,world", [(4194304, 8), (4194304, 3), (10, 4), (0, 2), (5, 8)])
def test_row_partition_properties(m, world):
    blocks = [row_partition(m, world, r) for r in range(world)]
    assert sum(c for _, c in blocks) == m
    nxt = 0
    for r0, c in blocks:
        if c:
            assert r0 == nxt
            nxt = r0 + c
    per = (m + world - 1) // world
    assert all(c <= per for _, c in blocks)
    with pytest.raises(ValueError):
        row_partition(m, world, world)
