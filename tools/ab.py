"""Interleaved A/B timing of shgemm tunables on the same inputs (robust to box-to-box clock drift):
each variant runs `rounds` times in round-robin; median ms, GB/s, TFLOP/s and cycles/stage."""
import sys, json, statistics, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg

def run(shape, variants, rounds=5, reps=5):
    m, k, n = shape
    A = shg.synth('gauss', 2, 0x100, m, k); Om = shg.gen_omega(k, n); Y = torch.empty((m, n), device='cuda')
    res = {name: [] for name, _ in variants}
    cyc = {}
    for name, tune in variants:
        pl = shg.plan(m, n, k, tune)
        prof = torch.zeros((pl['grid'], 16), dtype=torch.int64, device='cuda')
        t = dict(tune or {}); t['prof'] = prof.data_ptr()
        shg.shgemm(A, Om, out=Y, tune=t); torch.cuda.synchronize()
        cyc[name] = float(prof[:, 0].max() / prof[:, 11].max().clamp(min=1))
        cyc[name + '_ctas'] = int((prof[:, 0] > 0).sum())
        cyc[name + '_cycles'] = float(prof[:, 0].max())
    for _ in range(rounds):
        for name, tune in variants:
            for _ in range(2): shg.shgemm(A, Om, out=Y, tune=tune)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(reps): shg.shgemm(A, Om, out=Y, tune=tune)
            e.record(); torch.cuda.synchronize()
            res[name].append(s.elapsed_time(e) / reps)
    out = []
    for name, _ in variants:
        ms = statistics.median(res[name])
        out.append(dict(shape=shape, variant=name, ms=ms, gbs=(4.0*m*k+2.0*k*n+4.0*m*n)/ms/1e6, tflops=2.0*m*n*k/ms/1e9,
                        cyc_per_stage=cyc[name], spread=(max(res[name]) - min(res[name])) / ms,
                        ctas=cyc[name + '_ctas'], ghz_eff=cyc[name + '_cycles'] / ms / 1e6))
        print(json.dumps(out[-1]), flush=True)
    del A, Y; torch.cuda.empty_cache()
    return out

if __name__ == '__main__':
    allres = []
    for shape in [(1 << 21, 4096, 256), (32768, 32768, 16), (32768, 32768, 64), (32768, 32768, 128), (32768, 32768, 1024), (16384, 16384, 272)]:
        allres += run(shape, [('auto', None), ('pair_on', {'pair': 1}), ('pair_off', {'pair': 2})])
    json.dump(allres, open('gpurun_out/ab.json', 'w'), indent=1)
