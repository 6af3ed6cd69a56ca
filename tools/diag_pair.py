import sys, json, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
from tools.diag import SLOTS
m, k, n = 1 << 20, 4096, 256
A = shg.synth('gauss', 2, 0x100, m, k); Om = shg.gen_omega(k, n); Y = torch.empty((m, n), device='cuda')
for pair in (2, 1):
    for flags in (0, 3, 7):
        pl = shg.plan(m, n, k, {'pair': pair})
        prof = torch.zeros((pl['grid'], 16), dtype=torch.int64, device='cuda')
        tune = {'pair': pair, 'debug_flags': flags, 'prof': prof.data_ptr()}
        for _ in range(3): shg.shgemm(A, Om, out=Y, tune=tune)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); shg.shgemm(A, Om, out=Y, tune=tune); e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        pr = prof.double()
        for role, rows in (('leader/all', pr[0::2] if pair == 1 else pr), ('follower', pr[1::2] if pair == 1 else None)):
            if rows is None: continue
            st = rows[:, 11].mean()
            print(json.dumps(dict(pair=pair, flags=flags, role=role, ms=ms, clk_ghz=float(pr[:, 0].max()) / ms / 1e6,
                                  per_stage={SLOTS[i]: round(float(rows[:, i].mean() / st)) for i in range(11)})), flush=True)
