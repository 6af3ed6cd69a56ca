"""SHGEMM-TF32 vs SHGEMM-FP16 timing on the BASELINE shapes (interleaved rounds)."""
import sys, json, statistics, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg

def t_ms(fn, reps=5):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps

for m, k, n in [(1 << 21, 4096, 256), (32768, 32768, 64), (32768, 32768, 128), (32768, 32768, 1024), (16384, 16384, 272)]:
    A = shg.synth('gauss', 2, 0x100, m, k); Om = shg.gen_omega(k, n); Y = torch.empty((m, n), device='cuda')
    ws = {tc: torch.empty(max(1, shg.workspace_size(m, n, k, tc=tc)), dtype=torch.uint8, device='cuda') for tc in ('fp16', 'tf32')}
    res = {'fp16': [], 'tf32': []}
    for _ in range(3):
        for tc in ('fp16', 'tf32'):
            res[tc].append(t_ms(lambda: shg.shgemm(A, Om, out=Y, tc=tc, workspace=ws[tc])))
    for tc in ('fp16', 'tf32'):
        ms = statistics.median(res[tc])
        print(json.dumps(dict(m=m, k=k, n=n, tc=tc, ms=round(ms, 4), tflops=round(2.0 * m * n * k / ms / 1e9, 1),
                              gbs=round((4.0 * m * k + 2.0 * k * n + 4.0 * m * n) / ms / 1e6, 1),
                              plan=shg.plan(m, n, k, tc=tc))), flush=True)
    del A, Y, ws; torch.cuda.empty_cache()
