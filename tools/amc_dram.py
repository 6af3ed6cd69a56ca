"""One call per A-multicast variant on one shape (for ncu: dram__bytes_read.sum per launch).
usage: python tools/amc_dram.py M K N"""
import sys, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg

m, k, n = (int(x) for x in sys.argv[1:4])
A = shg.synth('gauss', 2, 0x100, m, k)
Om = shg.gen_omega(k, n)
Y = torch.empty((m, n), device='cuda')
for a_mcast in (1, 2, 4):
    try:
        shg.plan(m, n, k, {'a_mcast': a_mcast})
    except Exception:
        continue
    shg.shgemm(A, Om, out=Y, tune={'a_mcast': a_mcast})
    torch.cuda.synchronize()
    print('a_mcast', a_mcast, 'done', flush=True)
