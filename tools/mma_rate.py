import sys, json, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
L = shg.lib()
out = torch.zeros(148, device='cuda')
res = []
for n, ts, nacc in [(64,1,1),(64,1,2),(64,1,4),(128,1,1),(128,1,2),(128,1,3),(256,1,1),(64,0,1),(64,0,4),(128,0,1),(128,0,3),(256,0,1),(32,1,1),(32,1,4),(16,1,1),(16,1,8)]:
    st = L.shg_probe_mma_rate(n, 20000, ts, nacc << 3, shg._p(out), 148, shg._stream())
    torch.cuda.synchronize()
    c = float(out.mean())
    ideal = 128 * n / 256.0
    r = dict(n=n, ts=ts, nacc=nacc, status=st, cyc_per_mma=c, ideal=ideal, eff=ideal / c)
    print(json.dumps(r), flush=True); res.append(r)
json.dump(res, open('gpurun_out/mma_rate2.json', 'w'))
