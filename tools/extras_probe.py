import sys, json, torch
sys.path.insert(0, '.')
import bench, paper_2304_04612_b200 as shg
hbm, tc16, _, _ = bench.load_peaks()
which = sys.argv[1]
if which == "big":
    A = shg.synth("gauss", 2, 0x100, 4194304, 4096); torch.cuda.synchronize(); del A; torch.cuda.empty_cache()
if which == "keep":
    A = shg.synth("gauss", 2, 0x100, 4194304, 4096); torch.cuda.synchronize()
if which == "bench":   # the bench's sequence before its extras: cfg4 timed steps, then e2e
    A = shg.synth("gauss", 2, 0x100, 4194304, 4096); Om = shg.gen_omega(4096, 256); Y = torch.empty(4194304, 256, device="cuda")
    for _ in range(30): shg.shgemm(A, Om, out=Y)
    torch.cuda.synchronize()
    bench.measure_e2e(shg, torch, 4096, 256, steps=3)
    del A, Y; torch.cuda.empty_cache()
r = bench.measure_extras(shg, torch, hbm, tc16, 1.0)
print(which, json.dumps({k: round(v['ms'], 3) for k, v in r.items()}))
