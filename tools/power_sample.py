"""Power/clock samples (nvidia-smi, every ~100 ms) while the cfg4 SHGEMM runs back to back for ~5 s."""
import json
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

F = "power.draw,power.draw.instant,power.draw.average,power.limit,enforced.power.limit,clocks.sm,clocks_event_reasons.active,temperature.gpu"
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={F}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip()
        samples.append((time.time(), out))
        time.sleep(0.05)


m, k, n = 1 << 22, 4096, 256
A = shg.synth('gauss', 2, 0x100, m, k)
Om = shg.gen_omega(k, n)
Y = torch.empty((m, n), device='cuda')
torch.cuda.synchronize()
th = threading.Thread(target=sampler, daemon=True)
th.start()
time.sleep(1.0)
t0 = time.time()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(250):
    shg.shgemm(A, Om, out=Y)
e.record()
torch.cuda.synchronize()
t1 = time.time()
time.sleep(1.0)
stop.set()
th.join()
print(json.dumps({"fields": F, "ms_per_call": s.elapsed_time(e) / 250, "t_start": t0, "t_end": t1}))
for t, o in samples:
    print(json.dumps({"t": round(t - t0, 3), "s": o}))
