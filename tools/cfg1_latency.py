"""cfg1 (512 x 512 . 512 x 32) latency: per-call device time (events around each call), warm (back
to back) and cold (512 MiB L2 scrub between calls), for split-K choices and the Omega generator."""
import json
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

m = k = 512
n = 32
A = shg.synth("gauss", 2, 0x100, m, k)
Om = shg.gen_omega(k, n)
Y = torch.empty(m, n, device="cuda")
scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")


def per_call(fn, cold, reps=50):
    ts = []
    for i in range(reps + 5):
        if cold:
            scrub.fill_(i & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)


for name, tune in [("auto", None), ("sk1", {"split_k": 1}), ("sk2", {"split_k": 2}), ("sk4", {"split_k": 4})]:
    r = {"variant": name, "plan": shg.plan(m, n, k, tune)}
    r["warm_us"] = per_call(lambda: shg.shgemm(A, Om, out=Y, tune=tune, workspace=ws), False)
    r["cold_us"] = per_call(lambda: shg.shgemm(A, Om, out=Y, tune=tune, workspace=ws), True)
    print(json.dumps(r), flush=True)
print(json.dumps({"gen_omega_warm_us": per_call(lambda: shg.gen_omega(k, n), False),
                  "gen_omega_cold_us": per_call(lambda: shg.gen_omega(k, n), True)}))
