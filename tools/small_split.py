"""Small-problem split-K choice: cold device time per call (L2 scrubbed, events around a call queued
behind the scrub) for split_k 1/2/4/8 on small shapes; decides the auto plan's minimum k per split."""
import json
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")


def cold(fn, reps=40):
    ts = []
    for i in range(reps + 5):
        scrub.fill_(i & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)


for m, k, n in [(512, 512, 32), (512, 1024, 32), (512, 2048, 32), (1024, 1024, 64), (256, 4096, 16),
                (512, 4096, 32), (2048, 2048, 128)]:
    A = shg.synth("gauss", 2, 0x100, m, k)
    Om = shg.gen_omega(k, n)
    Y = torch.empty(m, n, device="cuda")
    r = {"m": m, "k": k, "n": n, "auto": shg.plan(m, n, k)["split_k"]}
    for sk in (1, 2, 4, 8):
        if sk > (k + 63) // 64:
            continue
        t = {"split_k": sk}
        r[f"sk{sk}_us"] = round(cold(lambda: shg.shgemm(A, Om, out=Y, tune=t, workspace=ws)), 2)
    print(json.dumps(r), flush=True)
