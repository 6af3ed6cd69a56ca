"""Critical-path diagnostics for the SHGEMM mainloop: per-role wait cycles (KParams::prof) and
ablations (debug_flags). Results are printed as JSON lines and saved to gpurun_out/diag_<tag>.json."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_04612_b200 as shg

SLOTS = ["total", "mma_acc_empty", "mma_hl_full", "mma_om_full", "split_a_full", "split_b_empty",
         "epi_acc_full", "prodA_a_empty", "prodB_b_empty", "split_busy", "epi_store", "stages"]


def t_ms(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def run(tag, shapes, flags_list=(0, 1, 2, 4, 3, 7), extra_tune=None):
    out = []
    for m, k, n in shapes:
        A = shg.synth("gauss", 2, 0x100, m, k)
        Om = shg.gen_omega(k, n, seed=0)
        Y = torch.empty((m, n), device="cuda")
        pl = shg.plan(m, n, k)
        prof = torch.zeros((pl["grid"], 16), dtype=torch.int64, device="cuda")
        for flags in flags_list:
            tune = {"debug_flags": flags}
            if extra_tune:
                tune.update(extra_tune)
            ms = t_ms(lambda: shg.shgemm(A, Om, out=Y, tune=tune))
            tune["prof"] = prof.data_ptr()
            shg.shgemm(A, Om, out=Y, tune=tune)
            torch.cuda.synchronize()
            pr = prof.double().mean(0).tolist()
            st = max(pr[11], 1.0)
            rec = {"m": m, "k": k, "n": n, "flags": flags, "ms": ms,
                   "gbs": (4.0 * m * k + 2.0 * k * n + 4.0 * m * n) / ms / 1e6,
                   "tflops": 2.0 * m * n * k / ms / 1e9,
                   "per_stage_cycles": {SLOTS[i]: pr[i] / st for i in range(11)}, "stages_per_cta": pr[11]}
            print(json.dumps(rec), flush=True)
            out.append(rec)
        del A, Y
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "d"
    shapes = [(1 << 20, 4096, 256), (32768, 32768, 64), (32768, 32768, 16), (32768, 32768, 1024)]
    res = run(tag, shapes)
    json.dump(res, open(f"gpurun_out/diag_{tag}.json", "w"), indent=1)
