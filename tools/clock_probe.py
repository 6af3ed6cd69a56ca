import sys, json, subprocess, threading, time, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
L = shg.lib()
def smi():
    r = subprocess.run(['nvidia-smi', '--query-gpu=clocks.sm,clocks.max.sm,clocks.applications.graphics,power.draw,power.limit,temperature.gpu,clocks_event_reasons.active', '--format=csv,noheader'], capture_output=True, text=True)
    return r.stdout.strip()
print('idle:', smi())
out = torch.zeros(148, device='cuda')
for iters in (200000, 2000000):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); L.shg_probe_mma_rate(256, iters, 1, 8, shg._p(out), 148, shg._stream()); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e); cyc = float(out.mean()) * iters
    print(json.dumps(dict(test='mma_probe', iters=iters, ms=ms, cycles=cyc, clock_ghz=cyc / ms / 1e6, smi=smi())), flush=True)
# shgemm with everything but TMA skipped (flags 7) and full (flags 0): cycles/time
for flags in (7, 0):
    m, k, n = 1 << 21, 4096, 256
    A = shg.synth('gauss', 2, 0x100, m, k); Om = shg.gen_omega(k, n); Y = torch.empty((m, n), device='cuda')
    pl = shg.plan(m, n, k); prof = torch.zeros((pl['grid'], 16), dtype=torch.int64, device='cuda')
    tune = {'prof': prof.data_ptr(), 'debug_flags': flags}
    for _ in range(2): shg.shgemm(A, Om, out=Y, tune=tune)
    torch.cuda.synchronize()
    for reps in (1, 20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps): shg.shgemm(A, Om, out=Y, tune=tune)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        cyc = float(prof[:, 0].max())
        print(json.dumps(dict(test=f'shgemm_flags{flags}', reps=reps, ms=ms, cycles=cyc, clock_ghz=cyc / ms / 1e6, gbs=4.0*m*k/ms/1e6, smi=smi())), flush=True)
    del A, Y; torch.cuda.empty_cache()
# plain torch copy for reference (GB/s)
x = torch.empty(1 << 30, dtype=torch.float32, device='cuda'); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): y.copy_(x)
e.record(); torch.cuda.synchronize()
print(json.dumps(dict(test='torch_copy', gbs=2 * 4.0 * (1 << 30) * 10 / s.elapsed_time(e) / 1e6, smi=smi())))
