"""A/B of the Omega generator between two package trees (e.g. HEAD built under abold/ vs the working
tree): each round runs one process per tree, interleaved; prints one JSON line per (tree, round).

usage: python tools/ab_gen.py <rootA> <rootB> [rounds]
Times gen_omega_tiled(2^20, 64) (cfg3's Omega per mode), gen_omega(4096, 256) (cfg4), and project() on
the cfg3 tensor (1024^3, n = 64) per mode with the separate generator and with in-kernel Omega."""
import json
import subprocess
import sys

CHILD = r'''
import json, sys, torch
sys.path.insert(0, ".")
import paper_2304_04612_b200 as shg

def t_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

K = 1 << 20
out = {"gen_tiled_2e20x64_ms": t_ms(lambda: shg.gen_omega_tiled(K, 64)),
       "gen_rowmajor_4096x256_ms": t_ms(lambda: shg.gen_omega(4096, 256))}
T = shg.synth("gauss", 1, 0x102, 1024, 1024 * 1024).view(1024, 1024, 1024)
ws = torch.empty(max(shg.project_workspace_size([1024] * 3, md, 64) for md in range(3)), dtype=torch.uint8,
                 device="cuda")
W = torch.empty(1024, 64, device="cuda")
for gen, tag in ((0, "separate"), (1, "inkernel"), (3, "inkernel_warp")):
    shg.lib().shg_set_inkernel_omega(gen)
    for mode in range(3):
        out[f"project_mode{mode}_{tag}_ms"] = t_ms(lambda: shg.project(T, mode, 64, workspace=ws, out=W), reps=10)
shg.lib().shg_set_inkernel_omega(0)
print(json.dumps(out))
'''


def main():
    roots = sys.argv[1:3]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    for r in range(rounds):
        for root in roots:
            res = subprocess.run([sys.executable, "-c", CHILD], cwd=root, capture_output=True, text=True)
            line = res.stdout.strip().splitlines()[-1] if res.stdout.strip() else None
            rec = {"root": root, "round": r}
            if res.returncode == 0 and line:
                rec.update(json.loads(line))
            else:
                rec["error"] = res.stderr[-2000:]
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
