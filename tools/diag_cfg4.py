"""cfg4 vs cfg5 per-stage cycles and effective SM clock (cycles / time)."""
import sys, json, subprocess, threading, time, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
from tools.diag import SLOTS

def clocks(stop, out):
    while not stop.is_set():
        r = subprocess.run(['nvidia-smi', '--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active', '--format=csv,noheader,nounits'], capture_output=True, text=True)
        out.append(r.stdout.strip()); time.sleep(0.05)

for (m, k, n, reps) in [(4194304, 4096, 256, 10), (1 << 20, 4096, 256, 20), (148 * 128 * 4, 32768, 256, 20), (32768, 32768, 256, 40)]:
    A = shg.synth('gauss', 2, 0x100, m, k)
    Om = shg.gen_omega(k, n, seed=0)
    Y = torch.empty((m, n), device='cuda')
    pl = shg.plan(m, n, k)
    prof = torch.zeros((pl['grid'], 16), dtype=torch.int64, device='cuda')
    tune = {'prof': prof.data_ptr()}
    for _ in range(3): shg.shgemm(A, Om, out=Y, tune=tune)
    torch.cuda.synchronize()
    st, samples = threading.Event(), []
    th = threading.Thread(target=clocks, args=(st, samples)); th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): shg.shgemm(A, Om, out=Y, tune=tune)
    e.record(); torch.cuda.synchronize(); st.set(); th.join()
    ms = s.elapsed_time(e) / reps
    pr = prof.double()
    tot = pr[:, 0]
    stages = pr[:, 11]
    rec = dict(m=m, k=k, n=n, ms=ms, gbs=(4.0*m*k + 2*k*n + 4.0*m*n)/ms/1e6, plan=pl,
               cycles_max=float(tot.max()), cycles_mean=float(tot.mean()), eff_clock_ghz=float(tot.max())/ms/1e6,
               stages_per_cta_max=float(stages.max()), cyc_per_stage=float(tot.max()/stages.max()),
               per_stage={SLOTS[i]: float(pr[:, i].mean() / stages.mean()) for i in range(11)},
               smi=samples[len(samples)//2] if samples else None)
    print(json.dumps(rec), flush=True)
    del A, Y; torch.cuda.empty_cache()
