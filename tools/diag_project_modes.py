"""project() per mode on the cfg3 tensor, in-kernel vs separate Omega, with the fallback counter (diagnostic)."""
import sys, json, torch
sys.path.insert(0, ".")
import paper_2304_04612_b200 as shg
T = shg.synth("gauss", 1, 0x102, 1024, 1024 * 1024).view(1024, 1024, 1024)
ws = torch.empty(max(shg.project_workspace_size([1024] * 3, md, 64) for md in range(3)), dtype=torch.uint8, device="cuda")
W = torch.empty(1024, 64, device="cuda")
def t_ms(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for rnd in range(3):
    for gen in (1, 0):
        shg.set_inkernel_omega(gen)
        for mode in range(3):
            h0 = shg.inkernel_omega_fallbacks()
            ms = t_ms(lambda: shg.project(T, mode, 64, workspace=ws, out=W))
            print(json.dumps(dict(rnd=rnd, gen=gen, mode=mode, ms=round(ms, 4), fallbacks=shg.inkernel_omega_fallbacks() - h0,
                                  plan=shg.plan(1024, 64, 1 << 20) if mode == 0 else None)), flush=True)
