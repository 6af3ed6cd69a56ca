import sys, json, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
L = shg.lib()
out = torch.zeros(148, device='cuda')
for n in (64, 128, 256):
    for ts in (1, 0):
        st = L.shg_probe_mma2_rate(n, 20000, ts, shg._p(out), 74, shg._stream())
        torch.cuda.synchronize()
        c = float(out[:74].mean())
        ideal = 128 * n / 256.0   # per-SM cycles for 128 x n x 16 at 4096 MAC/clk
        print(json.dumps(dict(cta_group=2, n=n, ts=ts, status=st, cyc_per_mma=c, ideal_per_sm=ideal, eff=ideal / c)), flush=True)
