"""Effective SM clock (clock64 cycles / time) of cfg4 under ablations, each after a 1 s cool-down
and run for ~1 s so the power controller settles."""
import sys, json, time, subprocess, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
m, k, n = 1 << 21, 4096, 256
A = shg.synth('gauss', 2, 0x100, m, k); Om = shg.gen_omega(k, n); Y = torch.empty((m, n), device='cuda')
pl = shg.plan(m, n, k); prof = torch.zeros((pl['grid'], 16), dtype=torch.int64, device='cuda')
CASES = [(0, 'full'), (8, 'no_omega_tma'), (16, 'omega_const_tile'), (32, 'a_const_kblock'), (48, 'both_const'),
         (1, 'no_promotion_loads'), (2, 'no_split_math'), (3, 'no_split_no_promo'), (4, 'no_mma'), (0, 'full_again')]
for flags, name in CASES:
    time.sleep(1.0)
    tune = {'prof': prof.data_ptr(), 'debug_flags': flags}
    t0 = time.time(); reps = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 1.0:
        for _ in range(10): shg.shgemm(A, Om, out=Y, tune=tune)
        reps += 10
        torch.cuda.synchronize()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    cyc = float(prof[:, 0].max())
    smi = subprocess.run(['nvidia-smi', '--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active', '--format=csv,noheader'], capture_output=True, text=True).stdout.strip()
    print(json.dumps(dict(case=name, flags=flags, ms=ms, clock_ghz=cyc / ms / 1e6, cyc=cyc, gbs=4.0 * m * k / ms / 1e6, smi=smi)), flush=True)
