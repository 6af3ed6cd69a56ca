"""Short-wide A (rows MiB apart): time shgemm vs padded leading dimension and row length, to tell
DRAM channel/page effects from pipeline effects (cfg3 mode-0 unfolding, 1024 x 2^20)."""
import sys, json, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg

def t_ms(fn, reps=5):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps

n = 64
buf = torch.empty(1024 * ((1 << 20) + 4096) + 4096, device='cuda')
for m, k in [(1024, 1 << 20), (2048, 1 << 19), (4096, 1 << 18), (8192, 1 << 17), (16384, 1 << 16), (65536, 1 << 14)]:
    Om = shg.gen_omega(k, n)
    pads = [0, 32, 64, 256, 1024] if m <= 2048 else [0, 64]
    for pad in pads:
        lda = k + pad
        A = buf[: m * lda].view(m, lda)
        A.normal_()
        Av = A[:, :k]
        for name, tune in [('auto', None), ('il_on', {'interleave': 1}), ('il_off', {'interleave': 2})]:
            pl = shg.plan(m, n, k, tune)
            ms = t_ms(lambda: shg.shgemm(Av, Om, tune=tune))
            print(json.dumps(dict(m=m, k=k, pad=pad, variant=name, split_k=pl['split_k'], ms=round(ms, 4),
                                  gbs=round(4.0 * m * k / ms / 1e6, 1))), flush=True)
    del Om
