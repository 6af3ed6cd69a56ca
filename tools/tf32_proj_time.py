import sys, json, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
T = shg.synth('gauss', 1, 0x102, 1024, 1024 * 1024).view(1024, 1024, 1024)
def t_ms(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize(); s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
ws = torch.empty(max(shg.project_workspace_size([1024]*3, md, 64, tc="tf32") for md in range(3)), dtype=torch.uint8, device='cuda')
print(json.dumps({f"tf32_mode{md}": t_ms(lambda: shg.project(T, md, 64, workspace=ws, tc="tf32")) for md in range(3)}))
