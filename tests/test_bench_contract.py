"""bench.py keeps the driver's contract: one JSON line with the required keys. The reference arm
(the CPU oracle) runs here; the GPU arm on a B200 (marked gpu) with a short cfg1 run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e"]


def run_bench(*args, timeout=600):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "1")
    for key in REQUIRED:
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"] == "cfg1"


@pytest.mark.gpu
def test_gpu_arm_contract():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench("--config", "cfg1", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    for key in REQUIRED + ["roofline", "gpu_launches", "clocks"]:
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] >= 5 * 2
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] <= 1.05 and r["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_gpus_flag_spawns_ranks_gloo():
    """`bench.py --gpus 2` without WORLD_SIZE (the driver's form) re-launches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1): rank 0 prints one line with n_gpus == 2 and the rows of both
    shards (SURVEY §8e row partition) summed over the process group."""
    env_ws = os.environ.pop("WORLD_SIZE", None)
    try:
        d = run_bench("--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3", timeout=300)
    finally:
        if env_ws is not None:
            os.environ["WORLD_SIZE"] = env_ws
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert d["rows_covered"] == d["config"]["m"] == 4194304
    assert d["config"]["rows_per_gpu"] == 2097152 and d["max_rank_plus_one"] == 2


def test_row_partition_covers_rows_once():
    sys.path.insert(0, ROOT)
    import bench
    for m in (1, 7, 512, 4194304, 4194305):
        for g in (1, 2, 3, 4, 8):
            spans = [bench.row_partition(m, g, r) for r in range(g)]
            covered = []
            for per, row0, rows in spans:
                covered.extend(range(row0, row0 + rows)) if m < 10000 else covered.append((row0, rows))
            if m < 10000:
                assert covered == list(range(m))
            else:
                assert sum(r for _, r in covered) == m
                assert all(covered[i][0] + covered[i][1] == covered[i + 1][0] for i in range(g - 1) if covered[i + 1][1])


@pytest.mark.gpu
def test_bench_nccl_plumbing_one_rank():
    """The NCCL path of the multi-rank bench (process group on the GPU, barrier, MAX all-reduce of the
    timed region, all-gather of the per-rank Omega CRC) on a one-GPU box: torchrun with one rank and
    SHG_BENCH_FORCE_DIST=1."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, SHG_BENCH_FORCE_DIST="1")
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--config", "cfg5n64", "--steps", "3", "--warmup", "3", "--no-extras", "--no-cpu-baseline",
                          "--no-e2e"], capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    d = json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])
    assert d["config"]["dist_backend"] == "nccl" and d["n_gpus"] == 1
    assert d["omega_identical_on_all_ranks"] is True and d["value"] > 0
