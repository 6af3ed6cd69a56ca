import sys, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
m = k = 32768
A = shg.synth('gauss', 2, 0x101, m, k)
for n in (512, 1024):
    Om = shg.gen_omega(k, n)
    Y = torch.empty((m, n), device='cuda')
    for mc in (0, 144):
        t = {'max_ctas': mc} if mc else None
        for _ in range(2):
            shg.shgemm(A, Om, out=Y, tune=t)
        torch.cuda.synchronize()
