"""Steady-state A/B of shgemm tunables under the 1000 W cap: per variant a block of back-to-back calls
(>= block_s seconds, preceded by a heating block of the same variant), blocks interleaved ABCABC...,
per-call event times (median of the block) and the SM clock / power sampled by NVML during the block.
usage: python tools/ab_steady.py OUT.json 'JSON variants [[name, tune], ...]' MxKxN [MxKxN ...]"""
import sys, json, time, statistics, threading, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg

try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:
    pynvml = None

VARIANTS = [('off', {'a_mcast': 1}), ('amc2', {'a_mcast': 2}), ('amc4', {'a_mcast': 4})]


def sample(stop, out):
    while not stop.is_set():
        if pynvml:
            out.append((pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(_h) / 1000.0))
        time.sleep(0.02)


def block(A, Om, Y, t, ncalls):
    evs = []
    for _ in range(ncalls):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        shg.shgemm(A, Om, out=Y, tune=t)
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in evs]


def run(m, k, n, rounds=3, block_s=1.5):
    A = shg.synth('gauss', 2, 0x100, m, k)
    Om = shg.gen_omega(k, n)
    Y = torch.empty((m, n), device='cuda')
    vs = []
    for name, t in VARIANTS:
        try:
            pl = shg.plan(m, n, k, t)
        except Exception:
            continue
        vs.append((name, t, pl))
    t0 = block(A, Om, Y, vs[0][1], 5)
    ncalls = max(20, int(block_s * 1e3 / statistics.median(t0)))
    res = {name: [] for name, _, _ in vs}
    clk = {name: [] for name, _, _ in vs}
    for r in range(rounds):
        for name, t, _ in vs:
            block(A, Om, Y, t, ncalls)                # heat with this variant
            stop, smp = threading.Event(), []
            th = threading.Thread(target=sample, args=(stop, smp))
            th.start()
            ts = block(A, Om, Y, t, ncalls)
            stop.set()
            th.join()
            res[name].append(statistics.median(ts))
            clk[name] += smp
    out = []
    for name, t, pl in vs:
        ms = statistics.median(res[name])
        mhz = statistics.median([c for c, _ in clk[name]]) if clk[name] else None
        w = statistics.median([p for _, p in clk[name]]) if clk[name] else None
        out.append(dict(m=m, k=k, n=n, variant=name, tune=t, a_mcast=pl['a_mcast'], ms=ms, per_round=res[name],
                        tflops=2.0 * m * n * k / ms / 1e9, sm_mhz=mhz, power_w=w, calls_per_block=ncalls))
        print(json.dumps(out[-1]), flush=True)
    del A, Y
    torch.cuda.empty_cache()
    return out


if __name__ == '__main__':
    outfile = sys.argv[1]
    VARIANTS[:] = [tuple(v) for v in json.loads(sys.argv[2])]
    shapes = [tuple(int(x) for x in a.split('x')) for a in sys.argv[3:]]
    allres = []
    for m, k, n in shapes:
        allres += run(m, k, n)
    json.dump(allres, open(outfile, 'w'), indent=1)
