"""Sustained (power-capped) A/B of tunables: ~1 s of back-to-back calls per variant per round, 1 s rest,
3 interleaved rounds; median ms per call. Usage: python tools/ab_sustained.py"""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402


def run(m, k, n, variants, rounds=3):
    A = shg.synth('gauss', 2, 0x101, m, k)
    Om = shg.gen_omega(k, n)
    Y = torch.empty((m, n), device='cuda')
    res = {name: [] for name, _ in variants}
    for _ in range(rounds):
        for name, tune in variants:
            time.sleep(1.0)
            for _ in range(3):
                shg.shgemm(A, Om, out=Y, tune=tune)
            torch.cuda.synchronize()
            t0 = time.time()
            reps = 0
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            while reps < 2000:
                shg.shgemm(A, Om, out=Y, tune=tune)
                reps += 1
                if reps % 50 == 0:
                    torch.cuda.synchronize()
                    if time.time() - t0 > 1.0:
                        break
            e.record()
            torch.cuda.synchronize()
            res[name].append(s.elapsed_time(e) / reps)
    for name, tune in variants:
        ms = statistics.median(res[name])
        print(json.dumps({"m": m, "k": k, "n": n, "variant": name, "ms": ms, "tflops": 2.0 * m * n * k / ms / 1e9,
                          "gbs": (4.0 * m * k + 2.0 * k * n + 4.0 * m * n) / ms / 1e6,
                          "plan": shg.plan(m, n, k, tune)}), flush=True)
    del A, Y
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for n in (128, 192, 256):
        run(32768, 32768, n, [("auto", None), ("pair_off", {"pair": 2}), ("pair_on", {"pair": 1})])
    run(32768, 32768, 64, [("auto", None), ("pair_on_bn128", {"pair": 1, "bn": 128})])
