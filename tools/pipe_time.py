"""Time RSVD (cfg2) and RP-HOSVD (cfg3) pipelines: SHGEMM projection vs SGEMM baseline, per line."""
import sys, json, torch
sys.path.insert(0, '.')
import numpy as np
import synth
import paper_2304_04612_b200 as shg
from paper_2304_04612_b200 import pipelines as pl

def best(fn, reps=3):
    out = None
    for _ in range(reps + 1):
        r = fn()
        if out is None or r['times_ms']['total'] < out['times_ms']['total']:
            out = r
    return out

N, p, s = 16384, 256, 16
A = synth.spectrum_matrix_torch(synth.spectrum('exp', N, p, 1e-2), seed=1)
for proj, gemm, fac in (('shgemm', 'tcec', 'gram'), ('shgemm', 'tcec', 'cusolver'), ('shgemm', 'sgemm', 'cusolver'),
                        ('sgemm', 'sgemm', 'cusolver')):
    r = best(lambda: pl.rsvd(A, p, s, seed=0, projection=proj, timing=True, gemm=gemm, factor=fac))
    e = pl.reconstruction_error(A, r['U'], r['S'], r['V'])
    print(json.dumps({'pipeline': 'rsvd_cfg2', 'projection': proj, 'gemm': gemm, 'factor': fac, 'times_ms': r['times_ms'], 'residual': e}), flush=True)
del A; torch.cuda.empty_cache()
T = torch.from_numpy(synth.alg3_tensor((1024, 1024, 1024), (64, 64, 64), pad=4, seed=1)).cuda()
for proj, gemm, fac in (('shgemm', 'tcec', 'gram'), ('shgemm', 'tcec', 'cusolver'), ('shgemm', 'sgemm', 'cusolver'),
                        ('sgemm', 'sgemm', 'cusolver')):
    r = best(lambda: pl.rp_hosvd(T, (64, 64, 64), seed=0, projection=proj, timing=True, gemm=gemm, factor=fac))
    e = pl.hosvd_error(T, r['core'], r['Q'])
    print(json.dumps({'pipeline': 'rphosvd_cfg3', 'projection': proj, 'gemm': gemm, 'factor': fac, 'times_ms': r['times_ms'], 'residual': e}), flush=True)
