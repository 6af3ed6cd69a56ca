"""Context for the power-bound claim: cuBLAS bf16 / fp16 GEMM on the SAME streaming shape as cfg4
(A 4,194,304 x 4096 in 16-bit, B 4096 x 256), sustained for ~2 s, with nvidia-smi clock/power
samples. cuBLAS does half the MMA work of SHGEMM (one product, not hi and lo) on half the A bytes."""
import json
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, '.')

samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw.instant",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append(out)
        time.sleep(0.1)


m, k, n = 1 << 22, 4096, 256
res = {}
for dt in (torch.bfloat16, torch.float16):
    A = torch.randn(m, k, device="cuda", dtype=dt)
    B = torch.randn(k, n, device="cuda", dtype=dt)
    C = torch.empty(m, n, device="cuda", dtype=dt)
    for _ in range(3):
        torch.matmul(A, B, out=C)
    torch.cuda.synchronize()
    time.sleep(1.0)
    samples.clear()
    stop.clear()
    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 200
    s.record()
    for _ in range(reps):
        torch.matmul(A, B, out=C)
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / reps
    clk = sorted(float(x.split(",")[0]) for x in samples[2:] if x)
    pw = sorted(float(x.split(",")[1]) for x in samples[2:] if x)
    res[str(dt)] = {"ms": ms, "tflops": 2.0 * m * n * k / ms / 1e9, "gbs": (2.0 * m * k + 2.0 * m * n) / ms / 1e6,
                    "sm_mhz_median": clk[len(clk) // 2] if clk else None, "power_w_median": pw[len(pw) // 2] if pw else None}
    del A, B, C
    torch.cuda.empty_cache()
print(json.dumps(res))
