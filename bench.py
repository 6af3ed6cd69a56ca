#!/usr/bin/env python
"""bench.py — SHGEMM random projection on B200 (BASELINE.json config 4, row-sharded).

One step = the whole hot path on this rank's row block: gen_omega_f16 (Omega regenerated from the
shared seed, no communication) + shgemm (TMA A stager, splitter, tcgen05 hi/lo MMAs, RN promotion,
epilogue). Inputs are resident in HBM before timing (A made in place by the counter-based
generator; 64 GiB / N per rank, far larger than L2, so no L2 flush is needed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl shgemm|reference] [--config cfg4|cfg5n256|...]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Prints ONE JSON line on rank 0 (keys per the driver contract, plus roofline and cpu_baseline).
--impl reference times the CPU oracle (oracle/, naive FP32 GEMM in C + its Omega generator) as
the reference arm, on a bounded sample of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SHGEMM TFLOP/s & % roofline at 1/2/4/8 B200; RSVD/RP-HOSVD time"
DATA_SEED, DATA_STREAM, OMEGA_SEED = 2, 0x100, 0

CONFIGS = {
    # name: (m_total, k, n, description)
    "cfg1": (512, 512, 32, "BASELINE config 1 shape: A 512x512 FP32 . Omega 512x32 FP16 (fits in L2: L2 flushed "
                           "between timed steps, only the steps timed)"),
    "cfg4": (4194304, 4096, 256, "BASELINE config 4: tall projection A 4,194,304x4096 FP32 . Omega 4096x256 FP16"),
    "cfg2proj": (16384, 16384, 272, "BASELINE config 2's projection (RSVD Alg 1 line 1): A 16384x16384 FP32 . "
                                    "Omega 16384x272 FP16"),
    "cfg5n64": (32768, 32768, 64, "BASELINE config 5 sweep point n=64 (m=k=32768)"),
    "cfg5n128": (32768, 32768, 128, "BASELINE config 5 sweep point n=128 (m=k=32768)"),
    "cfg5n256": (32768, 32768, 256, "BASELINE config 5 sweep point n=256 (m=k=32768)"),
    "cfg5n1024": (32768, 32768, 1024, "BASELINE config 5 sweep point n=1024 (m=k=32768)"),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    v = d.get(config)
    return None if v is None else float(v)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw.instant,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        # one nvidia-smi in loop mode (-lms: a sample every 50 ms) instead of a process per sample;
        # falls back to the per-sample loop if it yields nothing
        try:
            proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                     "--format=csv,noheader,nounits", "-lms", "50"],
                                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            proc = None
        if proc is not None:
            reader = threading.Thread(target=self._read, args=(proc,), daemon=True)
            reader.start()
            self._stop.wait()
            proc.terminate()
            try:
                proc.wait(timeout=5)
            except Exception:
                proc.kill()
            reader.join(timeout=5)
            if self.samples:
                return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def _read(self, proc):
        for line in proc.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 5 + i and s[5 + i].strip() == "Active"})
        pw = [float(s[3]) for s in self.samples if s[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w": statistics.median(pw) if pw else None}


def cpu_baseline(m, k, n, budget_s=30.0):
    """The oracle as it stands (naive FP32 GEMM, sequential fmaf over k, OpenMP over rows) on a
    bounded row sample of the same workload (grown until one timed sample takes ~8-10 s of CPU
    work); rate scaled to TFLOP/s."""
    import numpy as np
    import oracle
    om = oracle.omega_f16(k, n, seed=OMEGA_SEED)
    rows = 64
    t_used = 0.0
    elapsed, done = 0.0, 0
    while True:
        sample = np.arange(rows, dtype=np.int64) * max(1, m // rows)
        A = oracle.synth_rows("gauss", DATA_SEED, DATA_STREAM, sample, k)
        t0 = time.perf_counter()
        oracle.gemm_y32(A, om)
        dt = time.perf_counter() - t0
        elapsed, done = dt, rows
        t_used += dt
        if dt > budget_s / 4 or t_used > budget_s or rows >= m:
            break
        rows = min(m, int(rows * max(2.0, min(8.0, (budget_s / 3) / max(dt, 1e-3)))))
    flops = 2.0 * done * k * n
    return {"value": flops / elapsed / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{done} of {m} rows of A ({k}x{n} Omega), naive FP32 fmaf GEMM, {elapsed:.2f} s",
            **host_info()}


def run_reference(args, cfg_name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    m, k, n, desc = CONFIGS[cfg_name]
    # size one step so that warmup + steps fit in ~2-3 minutes
    rows = 2048
    A = oracle.synth_rows("gauss", DATA_SEED, DATA_STREAM, np.arange(rows, dtype=np.int64), k)
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        om = oracle.omega_f16(k, n, seed=OMEGA_SEED)
        oracle.gemm_y32(A, om)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    val = 2.0 * rows * k * n / t / 1e12
    cores = oracle.num_threads()
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg_name, "description": desc, "m": m, "k": k, "n": n,
                       "sample_rows_per_step": rows},
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                             "sample": f"{rows} rows of A per step + Omega generation, naive FP32 fmaf GEMM"},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


PIPELINES = {
    "rsvd_cfg2": "BASELINE config 2: Randomized SVD (Alg 1) of a 16384x16384 FP32 matrix (A_exp, s_p=1e-2), rank 256 + 16",
    "rphosvd_cfg3": "BASELINE config 3: RP-HOSVD (Alg 2) of a 1024^3 FP32 tensor (Alg 3, J=64, p=4, + 1e-2 N(0,1) noise), rank 64 per mode",
}


def run_pipeline(args):
    """Whole-pipeline device time (CUDA events per Alg line) with the SHGEMM projection vs the FP32
    SGEMM-baseline projection, median of --steps runs after --warmup."""
    import numpy as np
    import torch
    import synth
    from paper_2304_04612_b200 import pipelines as pl
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if args.config == "rsvd_cfg2":
        N, p, sov = 16384, 256, 16
        X = synth.spectrum_matrix_torch(synth.spectrum("exp", N, p, 1e-2), seed=1)
        run = lambda proj, gemm, fac: pl.rsvd(X, p, sov, seed=0, projection=proj, timing=True, gemm=gemm, factor=fac)
        err = lambda r: pl.reconstruction_error(X, r["U"], r["S"], r["V"])
        flops = 2.0 * N * N * (p + sov)
    else:
        # the noisy Alg-3 tensor (multilinear rank 60 + 1e-2 N(0,1)): an approximation-dominated
        # residual (~1e-2), so the residuals compared are not roundoff (reading c4-12 / c4-18)
        X = synth.alg3_tensor_torch((1024, 1024, 1024), (64, 64, 64), pad=4, seed=1, noise=1e-2)
        run = lambda proj, gemm, fac: pl.rp_hosvd(X, (64, 64, 64), seed=0, projection=proj, timing=True, gemm=gemm,
                                                  factor=fac)
        err = lambda r: pl.hosvd_error(X, r["core"], r["Q"])
        flops = 3 * 2.0 * X.numel() * 64
    res = {}
    # product: SHGEMM projection + TCEC-SGEMM for the other FP32 products (NEXT-2) + CholeskyQR2 /
    # Gram-eigh factorizations; the same with cuSOLVER QR/SVD; the paper's own configuration
    # (SHGEMM projection only); the FP32 SGEMM baseline pipeline
    variants = {"shgemm+tcec+gram": ("shgemm", "tcec", "gram"), "shgemm+tcec": ("shgemm", "tcec", "cusolver"),
                "shgemm": ("shgemm", "sgemm", "cusolver"), "sgemm": ("sgemm", "sgemm", "cusolver")}
    for name, (proj, gemm, fac) in variants.items():
        times, last = [], None
        for it in range(args.warmup + args.steps):
            last = run(proj, gemm, fac)
            if it >= args.warmup:
                times.append(last["times_ms"])
        tot = sorted(t["total"] for t in times)
        med = tot[len(tot) // 2]
        lines = {k: statistics.median(t[k] for t in times) for k in times[0] if k != "total"}
        res[name] = {"total_ms": med, "lines_ms": lines, "residual": err(last)}
    proj_key = [k for k in res["shgemm"]["lines_ms"] if "projection" in k][0]
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": res["shgemm+tcec+gram"]["total_ms"], "unit": "ms", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["shgemm+tcec+gram"]["total_ms"],
            "higher_is_better": False,
            "scaling": "none", "vs_baseline": None, "dtype": "f16*f16->f32 projection; TCEC f16 (FP32-accurate) other products; f64-Gram CholeskyQR2 / eigh",
            "data": "synthetic", "config": {"workload": args.config, "description": PIPELINES[args.config]},
            "pipeline": res, "speedup_vs_sgemm_pipeline": res["sgemm"]["total_ms"] / res["shgemm+tcec+gram"]["total_ms"],
            "speedup_projection_only_vs_sgemm_pipeline": res["sgemm"]["total_ms"] / res["shgemm"]["total_ms"],
            "projection_speedup": res["sgemm"]["lines_ms"][proj_key] / res["shgemm"]["lines_ms"][proj_key],
            "projection_tflops": flops / (res["shgemm"]["lines_ms"][proj_key] * 1e-3) / 1e12,
            "paper_context": "A100: 1.28x RSVD, 1.75x RP-HOSVD whole-pipeline speedups (P:12, P:786)"}), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """Re-run this command as N ranks (torch.distributed.run, 127.0.0.1 rendezvous); returns the
    launcher's exit code. Each rank binds LOCAL_RANK's GPU; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def row_partition(m_total: int, world: int, rank: int):
    """rank g owns rows [g*ceil(m/G), min(m, (g+1)*ceil(m/G)))."""
    per = (m_total + world - 1) // world
    row0 = min(m_total, rank * per)
    return per, row0, max(0, min(m_total, row0 + per) - row0)


def dry_run(args):
    """The multi-rank plumbing without the GPU: process group (gloo on CPU), row partition, the
    all-reduce(MAX) of a per-rank time, one line from rank 0."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    m_total, k, n, desc = CONFIGS[args.config]
    per, row0, m = row_partition(m_total, world, rank)
    rows = torch.tensor([float(m), float(rank + 1)])
    if world > 1:
        dist.init_process_group("gloo")
        dist.all_reduce(rows[:1], op=dist.ReduceOp.SUM)
        dist.all_reduce(rows[1:], op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "dry_run": True, "rows_covered": int(rows[0]),
                          "max_rank_plus_one": int(rows[1]),
                          "config": {"workload": args.config, "m": m_total, "k": k, "n": n, "rows_per_gpu": per}}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def host_info() -> dict:
    """CPU model, usable CPUs (sched_getaffinity) and host RAM of this box, for the CPU baseline."""
    info = {"affinity_cpus": len(os.sched_getaffinity(0)), "os_cpus": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["host_ram_gib"] = round(int(line.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return info


def oracle_sweep(budget_s: float = 1.5) -> dict:
    """SURVEY §8(d) oracle timing: the oracle as it stands (naive FP32 fmaf GEMM, OpenMP over rows;
    its Omega generator) on bounded row samples of configs 1, 2, 3 (one mode-n unfolding projection)
    and 5 (n = 16..4096); the full-config time is extrapolated linearly in m (rows are independent)
    and labelled so. Omega generation is timed on a sample of its elements and extrapolated the same way."""
    import numpy as np
    import oracle
    out = {"kind": "oracle", "cores": oracle.num_threads(), **host_info(), "configs": {}}
    # Omega generator rate (elements / s) on a 32768 x 64 sample
    t0 = time.perf_counter()
    oracle.omega_f16(32768, 64, seed=OMEGA_SEED)
    om_rate = 32768 * 64 / (time.perf_counter() - t0)
    out["omega_elements_per_s"] = om_rate

    def gemm_rate(m, k, n):
        om = oracle.omega_f16(k, n, seed=OMEGA_SEED) if k * n <= (1 << 26) else None
        if om is None:   # Omega too large to regenerate for a rate sample: time the first 2^26 / k rows of k
            raise ValueError
        rows0 = 8 * oracle.num_threads()        # >= 2 dynamic chunks of 4 rows per OpenMP thread
        rows, dt = min(m, rows0), 0.0
        while True:
            A = oracle.synth_rows("gauss", DATA_SEED, 0x101, np.arange(rows, dtype=np.int64), k)
            t = time.perf_counter()
            oracle.gemm_y32(A, om)
            dt = time.perf_counter() - t
            cap = min(m, max(rows0, min(4096, (1 << 26) // k)))   # <= 256 MiB of sampled A
            if dt > budget_s / 3 or rows >= cap:
                return rows, dt
            rows = min(cap, rows * max(2, int((budget_s / 3) / max(dt, 1e-4))))

    shapes = {"cfg1": (512, 512, 32), "cfg2_projection": (16384, 16384, 272),
              "cfg3_mode_projection": (1024, 1 << 20, 64)}
    for nn in (16, 32, 64, 128, 256, 512, 1024, 2048, 4096):
        shapes[f"cfg5_n{nn}"] = (32768, 32768, nn)
    for name, (m, k, n) in shapes.items():
        if k * n > (1 << 26):   # cfg5 n >= 4096: the GEMM rate is linear in n at fixed k; sample n = 2048
            rows, dt = gemm_rate(m, k, (1 << 26) // k)
            dt *= n / ((1 << 26) // k)
        else:
            rows, dt = gemm_rate(m, k, n)
        t_gemm = dt * m / rows
        t_gen = k * n / om_rate
        out["configs"][name] = {"m": m, "k": k, "n": n, "sample_rows": int(rows), "sample_s": dt,
                                "full_s_extrapolated": t_gemm + t_gen, "gemm_s_extrapolated": t_gemm,
                                "omega_gen_s_extrapolated": t_gen,
                                "tflops": 2.0 * m * k * n / (t_gemm + t_gen) / 1e12}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="shgemm", choices=["shgemm", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS) + sorted(PIPELINES))
    ap.add_argument("--tc", default="fp16", choices=["fp16", "tf32"],
                    help="SHGEMM-FP16 (default, the paper's headline kernel) or SHGEMM-TF32 (P:494-498)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the short per-config timings of BASELINE configs 2, 3 and 5 (single GPU, cfg4 runs)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU work: set up the ranks and the row partition and print the line's shape "
                         "(CPU test of the multi-rank launch)")
    ap.add_argument("--cpu-sweep", action="store_true",
                    help="time the CPU oracle on bounded samples of configs 1, 2, 3 and 5 (all n) and print "
                         "one JSON line (SURVEY §8(d) oracle timing)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` (the driver's form): re-launch this script with one rank per GPU
        # under torch.distributed.run; rank 0 prints the line for all N ranks
        sys.exit(spawn_ranks(args.gpus))
    if args.cpu_sweep:
        print(json.dumps(oracle_sweep()), flush=True)
        return
    if args.dry_run:
        dry_run(args)
        return

    if args.config in PIPELINES:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "pipeline modes have no reference arm"}))
            return
        run_pipeline(args)
        return
    if args.impl == "reference":
        run_reference(args, args.config)
        return

    import torch
    import paper_2304_04612_b200 as shg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    ndev = max(1, torch.cuda.device_count())
    local = int(os.environ.get("LOCAL_RANK", "0")) % ndev
    torch.cuda.set_device(local)
    dist = None
    backend = None
    # SHG_BENCH_FORCE_DIST=1 (under torchrun): set up the process group even for one rank, so the
    # NCCL plumbing (barrier, MAX all-reduce of the time, Omega CRC all-gather) runs on a 1-GPU box
    if world > 1 or (os.environ.get("SHG_BENCH_FORCE_DIST") == "1" and "WORLD_SIZE" in os.environ):
        import torch.distributed as dist
        # one rank per GPU over NCCL (the driver's launch); more ranks than GPUs (a functional test of
        # the sharded path on one device) cannot share a GPU under NCCL, so that case uses gloo.
        backend = "nccl" if world <= ndev else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    m_total, k, n, desc = CONFIGS[args.config]
    per, row0, m = row_partition(m_total, world, rank)

    A = shg.synth("gauss", DATA_SEED, DATA_STREAM, m, k, row0=row0)          # resident input
    Y = torch.empty((m, n), dtype=torch.float32, device="cuda")
    ldo = (k + 7) // 8 * 8
    om_buf = torch.empty((n, ldo), dtype=torch.float16, device="cuda")
    Om = om_buf[:, :k].t()
    stream = torch.cuda.current_stream()
    L = shg.lib()
    import ctypes
    tune = shg.Tune()
    tune.tc = shg.TCS[args.tc]
    # Omega generated straight into the column-major (K-major) layout the tensor cores stream, so the
    # step is two launches (no transpose pass; shgemm() also takes row-major Omega, bitwise the same Y)
    tune.omega_layout = shg.OMEGA_COL_MAJOR
    ws_bytes = shg.workspace_size(m, n, k, tc=args.tc)
    ws = torch.empty(max(1, ws_bytes), dtype=torch.uint8, device="cuda")

    def gen():
        shg._check(L.gen_omega_f16_ex(k, n, OMEGA_SEED, 0, 0, 0, k, shg._p(om_buf), ldo, shg.OMEGA_COL_MAJOR,
                                      shg._stream()), "gen_omega_f16_ex")

    def gemm():
        shg._check(L.shgemm_ex(m, n, k, shg._p(A), k, shg._p(om_buf), ldo, shg._p(Y), n, ctypes.byref(tune),
                               shg._p(ws), ws_bytes, None, shg._stream()), "shgemm_ex")

    def step():
        gen()
        gemm()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # inputs smaller than L2 (126 MB): the step is launch-latency bound, so it is replayed from CUDA
    # graphs (no host work between kernels), a 512 MiB buffer is written between timed steps (cold
    # L2) and only the steps are timed; otherwise the inputs are far larger than L2 and the steps run
    # back to back as direct launches
    flush = (4.0 * m * k) < 256e6
    scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if flush else None
    run_gen, run_gemm, graph_launches = gen, gemm, None
    if flush:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                step()
        torch.cuda.current_stream().wait_stream(side)
        g_gen, g_gemm = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        c0 = shg.launch_count()
        with torch.cuda.graph(g_gen):
            gen()
        with torch.cuda.graph(g_gemm):
            gemm()
        graph_launches = shg.launch_count() - c0          # library kernels per step (captured once)
        run_gen, run_gemm = g_gen.replay, g_gemm.replay
        torch.cuda.synchronize()
    # per-launch events for the dominant kernel (shgemm) and the Omega generator, on the launch stream
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    launches0 = shg.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        if flush:
            scrub.fill_(i & 0xFF)
        ev[i][0].record(stream)
        run_gen()
        ev[i][1].record(stream)
        run_gemm()
        ev[i][2].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = shg.launch_count() - launches0 if graph_launches is None else graph_launches * args.steps
    if dist:
        dist.barrier()
    clk = clocks.stop()
    # §8(e) check: every rank regenerated the identical Omega from the shared seed (CRC32 of its bits,
    # all-gathered; no Omega ever crossed between ranks)
    from paper_2304_04612_b200.shard import checksum_bits
    crc = checksum_bits(om_buf[:, :k])
    crcs = [crc]
    if dist:
        got = [None] * world
        dist.all_gather_object(got, crc)
        crcs = got
    total_ms = (sum(ev[i][0].elapsed_time(ev[i][2]) for i in range(args.steps)) if flush
                else t_start.elapsed_time(t_end))
    gemm_ms = statistics.mean(ev[i][1].elapsed_time(ev[i][2]) for i in range(args.steps))
    gen_ms = statistics.mean(ev[i][0].elapsed_time(ev[i][1]) for i in range(args.steps))
    if dist:
        t = torch.tensor([total_ms], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    flops_total = 2.0 * m_total * k * n
    value = flops_total / (ms_per_step * 1e-3) / 1e12
    fused = None
    if flush and world == 1:
        # the same step as ONE kernel: project(A, mode 0, n) with Omega generated
        # inside the mainloop (its stream_id 0 = gen_omega's), replayed from a CUDA graph like the
        # two-kernel step; reported beside it (latency-bound shapes only)
        try:
            fused = measure_fused_step(shg, torch, A, n, args.steps, scrub)
        except Exception as exc:  # noqa: BLE001
            fused = {"error": repr(exc)[:200]}

    hbm, tc16, tc16_sus, peak_src = load_peaks()
    # Roofline (north_star): min(P_FP16 / 2, AI x BW) with the BURST tensor peak (the
    # kernel is timed alone, one ~19-ms launch per step): HBM-bound for n <= 253, tensor-bound above.
    # cfg4 (AI = 120.5 flop/B) is HBM-bound, so `frac` = algorithmic bytes per launch / launch time /
    # measured HBM bandwidth. The sustained-peak tensor fraction is reported beside it, not as `frac`.
    tc_ratio = 0.5 if args.tc == "tf32" else 1.0            # TF32 tensor rate = half of FP16
    tc16, tc16_sus = tc16 * tc_ratio, tc16_sus * tc_ratio
    alg_bytes = 4.0 * m * k + 2.0 * k * n + 4.0 * m * n        # per launch, this rank
    achieved_gbs = alg_bytes / (gemm_ms * 1e-3) / 1e9
    ai = 2.0 * m * k * n / alg_bytes
    tc_ceiling = tc16 / 2.0                                     # two MMAs per product
    useful_tflops = 2.0 * m * k * n / (gemm_ms * 1e-3) / 1e12
    tc_ach = 4.0 * m * k * n / (gemm_ms * 1e-3) / 1e12         # tensor pipe: hi and lo MMAs
    bound = "hbm" if ai * hbm / 1e3 < tc_ceiling else "tensor"
    if bound == "hbm":
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s", "frac": achieved_gbs / hbm}
    else:
        roof = {"bound": "tensor", "achieved": tc_ach, "peak": tc16, "unit": "TFLOP/s", "frac": tc_ach / tc16}
    tag = args.config + ("" if args.tc == "fp16" else "_tf32")
    roof["traffic"] = ncu_traffic(tag if world == 1 else f"{tag}_g{world}")
    roof["peak_source"] = (f"{peak_src} (MEASURED_PEAKS.json): hbm_gbs; bf16_tflops (burst) for the bound"
                           + (" x 0.5 for TF32" if args.tc == "tf32" else ""))
    roof["kernel"] = "shgemm_sm100_kernel"
    roof["kernel_ms"] = gemm_ms
    roof["algorithmic_bytes_per_launch"] = alg_bytes
    roof["algorithmic_flops_per_launch"] = 2.0 * m * k * n
    roof["frac_of_min(tc_burst/2, AI*hbm)"] = useful_tflops / min(tc_ceiling, ai * hbm / 1e3)
    roof["frac_hbm"] = achieved_gbs / hbm
    roof["frac_tensor_burst"] = tc_ach / tc16
    roof["frac_tensor_sustained"] = tc_ach / tc16_sus       # context: the 1000 W cap
    # against the spec sheet (2250 TFLOP/s dense fp16/bf16, 8 TB/s HBM3e), for reference
    spec_tc = 2250.0 * tc_ratio
    roof["frac_spec_min(tc/2, AI*hbm)"] = useful_tflops / min(spec_tc / 2.0, ai * 8000.0 / 1e3)

    # e2e on EVERY rank at once (each GPU streams its own row sample over its own PCIe link from
    # pinned host memory): aggregate rows / max-over-ranks time
    e2e = None
    if not args.no_e2e:
        try:
            e2e = measure_e2e(shg, torch, k, n, steps=3, rank=rank, world=world, dist=dist, backend=backend)
        except Exception as exc:  # noqa: BLE001
            e2e = {"error": repr(exc)[:300]}
    out = None
    if rank == 0:
        # the other BASELINE configs first (device only, this workload's 64 GiB released: a resident
        # 64 GiB allocation measurably slows the strided unfolding reads), then e2e, then the CPU oracle
        # (its OpenMP threads would contend with the host side of the device timings)
        extras = None
        if not args.no_extras and world == 1 and args.config == "cfg4" and args.tc == "fp16":
            del A, Y
            torch.cuda.empty_cache()
            try:   # context only: never let it cost the headline line
                extras = measure_extras(shg, torch, hbm, tc16, 1.0)
            except Exception as exc:  # noqa: BLE001
                extras = {"error": repr(exc)[:300]}
                torch.cuda.empty_cache()
            ceil = (extras or {}).get("cublas_fp16_two_products_cfg4_bytes")
            if ceil and gemm_ms > 0:
                # context beside frac (DESIGN §5 "power-cap ceiling"): the same run's cuBLAS fp16 doing
                # SHGEMM's two products on its A bytes; shgemm time / that time is the share of the
                # power-capped ceiling the kernel reaches
                roof["power_cap_ceiling_ms"] = ceil["ms"]
                roof["frac_of_power_cap_ceiling"] = ceil["ms"] / gemm_ms
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(m_total, k, n)
            if args.config == "cfg4" and not args.no_extras:
                try:   # the oracle on configs 1, 2, 3, 5 (bounded samples, extrapolated)
                    sw = oracle_sweep()
                    cpu["configs"] = sw["configs"]
                    cpu["omega_elements_per_s"] = sw["omega_elements_per_s"]
                except Exception as exc:  # noqa: BLE001
                    cpu["configs_error"] = repr(exc)[:200]
        out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None,
               "dtype": ("f16*f16->f32 (FP32 A split to FP16 hi/lo in-kernel)" if args.tc == "fp16" else
                         "tf32*tf32->f32 (FP32 A split to TF32 hi/lo in-kernel; FP16 Omega widened exactly)"),
               "data": "synthetic",
               "config": {"workload": args.config, "description": desc, "m": m_total, "k": k, "n": n,
                          "rows_per_gpu": per, "parallelism": f"row-shard x{world} (no collective on the data path)",
                          "dist_backend": backend,
                          "l2": ("L2 flushed between timed steps (512 MiB write), steps replayed from CUDA graphs "
                                 "and timed alone" if flush else
                                 "inputs larger than L2 (A is %.1f GiB per GPU), no flush" % (4.0 * m * k / 2 ** 30)),
                          "kernel": "SHGEMM-FP16" if args.tc == "fp16" else "SHGEMM-TF32",
                          "plan": shg.plan(m, n, k, tc=args.tc)},
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
               "clocks": clk, "omega_gen_ms": gen_ms, "shgemm_ms": gemm_ms, "other_workloads": extras,
               "fused_single_launch_step": fused,
               "omega_crc32_per_rank": crcs, "omega_identical_on_all_ranks": len(set(crcs)) == 1,
               "gbs_algorithmic": achieved_gbs}
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def measure_fused_step(shg, torch, A, n, steps, scrub):
    """One step = project(A, 0, n, seed) with in-kernel Omega (one mainloop launch + a memset of its
    tile flags), CUDA-graph replay, L2 scrubbed between steps; per-step device time in us."""
    m, k = A.shape
    ws = torch.empty(shg.project_workspace_size([m, k], 0, n), dtype=torch.uint8, device="cuda")
    W = torch.empty((m, n), device="cuda")
    prev = shg.get_inkernel_omega()
    shg.set_inkernel_omega(True)
    try:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                shg.project(A, 0, n, seed=OMEGA_SEED, workspace=ws, out=W)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        c0 = shg.launch_count()
        with torch.cuda.graph(g):
            shg.project(A, 0, n, seed=OMEGA_SEED, workspace=ws, out=W)
        launches = shg.launch_count() - c0
    finally:
        shg.set_inkernel_omega(prev)
    torch.cuda.synchronize()
    ts = []
    for i in range(steps):
        scrub.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return {"us_per_step": statistics.mean(ts), "us_median": statistics.median(ts), "kernels_per_step": launches,
            "tflops": 2.0 * m * k * n / (statistics.mean(ts) * 1e-6) / 1e12,
            "step": "project(A, mode 0, n) with Omega generated in the mainloop (OMGEN)"}


def measure_extras(shg, torch, hbm, tc16_burst, tc_ratio, reps=10):
    """Short device timings (CUDA events, median of 5 rounds of `reps` calls; inputs >= 1 GiB, far
    larger than L2) of the hot path on the other BASELINE configs, each against its own roofline
    min(burst tensor / 2, AI x HBM): cfg2's projection (RSVD of 16384^2, n = 272), cfg3's project()
    of each mode (1024^3 tensor, n = 64, Omega generation included) and cfg5 at n = 64 and 1024."""
    import statistics as st

    def med_ms(fn, spread=False):
        # 5 rounds of `reps` back-to-back calls between two events (the host enqueues ahead of the
        # device, so host-side call overhead is not timed); median round, per call. Back to back the
        # GPU settles under the 1000 W cap within a few ms, so this is the SUSTAINED rate.
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / reps)
        return (st.median(ts), min(ts), max(ts)) if spread else st.median(ts)

    def iso_ms(fn, n_iso=7):
        # one call at a time after 50 ms idle (a 64 MiB scrub evicts the previous call's A from L2):
        # the BURST rate, i.e. a projection as one step of a pipeline sees it
        scrub = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        ts = []
        for _ in range(n_iso):
            scrub.zero_()
            torch.cuda.synchronize()
            time.sleep(0.05)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return st.median(ts)

    def roof(m, k, n, ms, iso=None):
        fl, by = 2.0 * m * k * n, 4.0 * m * k + 2.0 * k * n + 4.0 * m * n
        ceil = min(tc16_burst * tc_ratio / 2.0, fl / by * hbm / 1e3)
        d = {"ms": ms, "tflops": fl / ms / 1e9, "gbs": by / ms / 1e6, "frac_roofline": fl / ms / 1e9 / ceil,
             "bound": "tensor" if tc16_burst * tc_ratio / 2.0 < fl / by * hbm / 1e3 else "hbm"}
        if iso is not None:   # single call after idle: burst clocks
            d.update(ms_isolated=iso, frac_roofline_isolated=fl / iso / 1e9 / ceil)
        return d

    out = {}
    # a READ-ONLY HBM stream (reported beside the copy bandwidth of MEASURED_PEAKS.json):
    # the library's TMA-only probe streams a 4 GiB matrix into shared memory in the mainloop's tile
    # order (one 4-D box of 2 x 32 k x 128 rows per stage, no math)
    try:
        import ctypes
        L = shg.lib()
        buf = torch.empty(32768 * 32768, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")

        def tma_read():
            st = L.shg_probe_tma_read(ctypes.c_void_p(buf.data_ptr()), 32768, 32768, 32768, 2, 64, 128, 1, 148,
                                      ctypes.c_void_p(cnt.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            assert st == 0, st
        ms = med_ms(tma_read)
        out["hbm_read_only_probe"] = {"ms": ms, "gbs": 4.0 * 32768 * 32768 / ms / 1e6,
                                      "note": "shg_probe_tma_read: TMA-only read of 4 GiB (256 B per row visit), "
                                              "back to back; the HBM-bound kernels' GB/s can be read against it too"}
        del buf, cnt
        torch.cuda.empty_cache()
    except Exception as exc:  # noqa: BLE001
        out["hbm_read_only_probe"] = {"error": repr(exc)[:200]}
    # context for the power cap: cuBLAS bf16 on cfg4's own shape (one 16-bit product, half the A bytes)
    m4, k4, n4 = 4194304, 4096, 256
    Ab = torch.randn(m4, k4, device="cuda", dtype=torch.bfloat16)
    Bb = torch.randn(k4, n4, device="cuda", dtype=torch.bfloat16)
    Cb = torch.empty(m4, n4, device="cuda", dtype=torch.bfloat16)
    ms = med_ms(lambda: torch.matmul(Ab, Bb, out=Cb))
    out["cublas_bf16_cfg4_shape"] = {"ms": ms, "tensor_tflops": 2.0 * m4 * n4 * k4 / ms / 1e9,
                                     "note": "torch.matmul bf16, A 4194304x4096 . B 4096x256: ONE product on 16-bit A; "
                                             "SHGEMM's tensor work is two products on FP32 A (compare its 4mnk/t)"}
    del Ab, Bb, Cb
    torch.cuda.empty_cache()
    # the power-cap ceiling of SHGEMM's own work: cuBLAS fp16 doing BOTH products
    # on the same bytes as one GEMM, [A_hi | A_lo] (m x 2k FP16 = the 4mk bytes of FP32 A) times
    # [Omega; Omega] (2k x n): the tensor flops (4mnk) and A bytes of SHGEMM without its split and
    # RN promotion (and with a 2-byte output)
    A2 = torch.randn(m4, 2 * k4, device="cuda", dtype=torch.float16)
    B2 = torch.randn(2 * k4, n4, device="cuda", dtype=torch.float16)
    C2 = torch.empty(m4, n4, device="cuda", dtype=torch.float16)
    ms = med_ms(lambda: torch.matmul(A2, B2, out=C2))
    out["cublas_fp16_two_products_cfg4_bytes"] = {
        "ms": ms, "tensor_tflops": 4.0 * m4 * n4 * k4 / ms / 1e9, "useful_tflops_equiv": 2.0 * m4 * n4 * k4 / ms / 1e9,
        "gbs": (4.0 * m4 * k4 + 4.0 * k4 * n4 + 2.0 * m4 * n4) / ms / 1e6,
        "note": "torch.matmul fp16, (4194304 x 8192) . (8192 x 256): SHGEMM-FP16's 4mnk tensor flops on its 4mk "
                "A bytes, no split / promotion: the power-capped ceiling for the method on this box"}
    del A2, B2, C2
    torch.cuda.empty_cache()
    shapes = {"cfg2_projection": (16384, 16384, 272)}
    for nn in (16, 32, 64, 128, 256, 512, 1024, 2048, 4096):      # BASELINE config 5: the whole sweep
        shapes[f"cfg5_n{nn}"] = (32768, 32768, nn)
    A5 = None
    for name, (m, k, n) in shapes.items():
        if name.startswith("cfg5"):
            A5 = shg.synth("gauss", DATA_SEED, 0x101, m, k) if A5 is None else A5
            A = A5
        else:
            A = shg.synth("gauss", DATA_SEED, 0x101, m, k)
        Om = torch.empty((n, k), dtype=torch.float16, device="cuda").t()
        Y = torch.empty((m, n), device="cuda")
        fn = lambda: (shg.gen_omega(k, n, seed=OMEGA_SEED, out=Om), shg.shgemm(A, Om, out=Y))
        ms = med_ms(fn)
        out[name] = dict(roof(m, k, n, ms, iso_ms(fn)), m=m, k=k, n=n, step="gen_omega_f16 + shgemm",
                         a_mcast=shg.plan(m, n, k)["a_mcast"])
        if name in ("cfg2_projection", "cfg5_n256", "cfg5_n1024", "cfg5_n4096"):
            # the power-capped ceiling of the method's own tensor work on this shape (as for cfg4):
            # cuBLAS fp16 doing both products, [A_hi | A_lo] (m x 2k) . [Omega; Omega] (2k x n)
            A2 = torch.randn(m, 2 * k, device="cuda", dtype=torch.float16)
            B2 = torch.randn(2 * k, n, device="cuda", dtype=torch.float16)
            C2 = torch.empty(m, n, device="cuda", dtype=torch.float16)
            cms = med_ms(lambda: torch.matmul(A2, B2, out=C2))
            out[name]["power_cap_ceiling_ms"] = cms
            out[name]["frac_of_power_cap_ceiling"] = cms / ms
            del A2, B2, C2
            torch.cuda.empty_cache()
        if out[name]["a_mcast"] > 1 and n <= 1024:
            # the same step with A multicast off (per-pair A loads; DESIGN.md §5 "A read once")
            fn_off = lambda: (shg.gen_omega(k, n, seed=OMEGA_SEED, out=Om), shg.shgemm(A, Om, out=Y, tune={"a_mcast": 1}))
            out[name]["a_mcast_off"] = roof(m, k, n, med_ms(fn_off))
        del A, Om, Y
        torch.cuda.empty_cache()
    del A5
    torch.cuda.empty_cache()
    T = shg.synth("gauss", 1, 0x102, 1024, 1024 * 1024).view(1024, 1024, 1024)
    ws = torch.empty(max(shg.project_workspace_size([1024] * 3, md, 64) for md in range(3)), dtype=torch.uint8,
                     device="cuda")
    W = torch.empty((1024, 64), device="cuda")
    for mode in range(3):
        fn = lambda: shg.project(T, mode, 64, workspace=ws, out=W)
        ms, lo, hi = med_ms(fn, spread=True)
        out[f"cfg3_project_mode{mode}"] = dict(roof(1024, 1 << 20, 64, ms, iso_ms(fn)), m=1024, k=1 << 20, n=64,
                                               ms_min=lo, ms_max=hi, step="project() incl. Omega generation")
    del T, ws, W
    torch.cuda.empty_cache()
    try:
        out.update(measure_pipelines(torch))
    except Exception as exc:  # noqa: BLE001
        out["pipelines_error"] = repr(exc)[:300]
        torch.cuda.empty_cache()
    return out


def measure_pipelines(torch, reps=3):
    """The metric's "RSVD/RP-HOSVD time": configs 2 and 3 end to end on the device (CUDA events per
    Alg line), the product pipeline (SHGEMM projection, TCEC-SGEMM products, CholeskyQR2 / Gram-eigh)
    against the FP32 SGEMM + cuSOLVER baseline; median of `reps` runs after one warm-up each."""
    import statistics as st
    import synth
    from paper_2304_04612_b200 import pipelines as pl

    def best(fn):
        fn()
        runs = [fn() for _ in range(reps)]
        return sorted(runs, key=lambda r: r["times_ms"]["total"])[len(runs) // 2]

    out = {}
    X = synth.spectrum_matrix_torch(synth.spectrum("exp", 16384, 256, 1e-2), seed=1)
    prod = best(lambda: pl.rsvd(X, 256, 16, seed=0, timing=True, gemm="tcec", factor="gram"))
    base = best(lambda: pl.rsvd(X, 256, 16, seed=0, projection="sgemm", timing=True))
    out["rsvd_cfg2_pipeline"] = {"ms": prod["times_ms"]["total"], "lines_ms": prod["times_ms"],
                                 "sgemm_baseline_ms": base["times_ms"]["total"],
                                 "speedup": base["times_ms"]["total"] / prod["times_ms"]["total"],
                                 "residual": pl.reconstruction_error(X, prod["U"], prod["S"], prod["V"]),
                                 "residual_baseline": pl.reconstruction_error(X, base["U"], base["S"], base["V"])}
    del X, prod, base
    torch.cuda.empty_cache()
    T = synth.alg3_tensor_torch((1024, 1024, 1024), (64, 64, 64), pad=4, seed=1, noise=1e-2)
    prod = best(lambda: pl.rp_hosvd(T, (64, 64, 64), seed=0, timing=True, gemm="tcec", factor="gram"))
    base = best(lambda: pl.rp_hosvd(T, (64, 64, 64), seed=0, projection="sgemm", timing=True))
    out["rphosvd_cfg3_pipeline"] = {"ms": prod["times_ms"]["total"], "lines_ms": prod["times_ms"],
                                    "sgemm_baseline_ms": base["times_ms"]["total"],
                                    "speedup": base["times_ms"]["total"] / prod["times_ms"]["total"],
                                    "residual": pl.hosvd_error(T, prod["core"], prod["Q"]),
                                    "residual_baseline": pl.hosvd_error(T, base["core"], base["Q"])}
    del T, prod, base
    torch.cuda.empty_cache()
    return out


def measure_e2e(shg, torch, k, n, steps=3, rank=0, world=1, dist=None, backend=None):
    """Same metric through the C ABI with HOST buffers: each step copies this rank's row sample of A
    from pinned host memory to its device, projects it (shgemm_host streams overlapped chunks) and
    copies Y back; host<->device copies are inside the timed region. All ranks run at once (a
    barrier before the timed steps); value = all ranks' rows / the max-over-ranks time."""
    rows = 262144 if k <= 4096 else max(128, (1 << 30) // (4 * k))
    A_h = shg.synth("gauss", DATA_SEED, DATA_STREAM, rows, k, row0=rank * rows).cpu().pin_memory()
    Y_h = torch.empty((rows, n), dtype=torch.float32).pin_memory()
    ws = torch.empty(shg.host_workspace_size(n, k), dtype=torch.uint8, device="cuda")

    def step():
        Om = shg.gen_omega(k, n, seed=OMEGA_SEED)
        shg.shgemm_host(A_h, Om, Y_h, workspace=ws)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        step()
    e.record()
    torch.cuda.synchronize()
    dt = s.elapsed_time(e) / 1e3 / steps
    if dist:
        t = torch.tensor([dt], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    return {"value": 2.0 * world * rows * k * n / dt / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": world * rows * k * 4, "d2h_bytes_per_step": world * rows * n * 4,
            "rows_per_step": world * rows, "ms_per_step": dt * 1e3, "ranks": world,
            "api": "shgemm_host (C ABI, pinned host A/Y, overlapped chunk streaming), every rank"}


if __name__ == "__main__":
    main()
