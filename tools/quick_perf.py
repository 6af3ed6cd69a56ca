"""Scratch timing of shgemm on a few shapes (CUDA events); not the bench contract."""
import sys, json, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg

def t_ms(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

res = []
shapes = [(4194304, 4096, 256), (32768, 32768, 16), (32768, 32768, 64), (32768, 32768, 128), (32768, 32768, 256),
          (32768, 32768, 512), (32768, 32768, 1024), (16384, 16384, 272), (1024, 1 << 20, 64), (512, 512, 32)]
if len(sys.argv) > 1: shapes = shapes[:int(sys.argv[1])]
for m, k, n in shapes:
    A = shg.synth('gauss', 2, 0x100, m, k)
    Om = shg.gen_omega(k, n, seed=0)
    Y = torch.empty((m, n), device='cuda')
    ms = t_ms(lambda: shg.shgemm(A, Om, out=Y), reps=5 if m*k > 1e10 else 20)
    fl = 2.0*m*n*k/ms/1e9
    gbs = (4.0*m*k + 2.0*k*n + 4.0*m*n)/ms/1e6
    r = dict(m=m, k=k, n=n, ms=ms, tflops=fl, gbs=gbs, plan=shg.plan(m, n, k))
    print(json.dumps(r), flush=True); res.append(r)
    del A, Y; torch.cuda.empty_cache()
json.dump(res, open('gpurun_out/quick_perf.json', 'w'), indent=1)
