import sys, json, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
T = shg.synth('gauss', 1, 0x102, 1024, 1024 * 1024).view(1024, 1024, 1024)
def t_ms(fn, reps=5):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / reps
ws = torch.empty(max(shg.project_workspace_size([1024]*3, md, 64) for md in range(3)), dtype=torch.uint8, device='cuda')
for mode in range(3):
    ms = t_ms(lambda: shg.project(T, mode, 64, workspace=ws))
    print(json.dumps(dict(mode=mode, ms=ms, gbs=4.0 * 2**30 / ms / 1e6)), flush=True)
Om = shg.gen_omega(1 << 20, 64)
A = T.view(1024, -1)
for sk in (0, 9, 18, 36):
    ms = t_ms(lambda: shg.shgemm(A, Om, tune={'split_k': sk} if sk else None))
    print(json.dumps(dict(mode='0-shgemm', split_k=sk, plan=shg.plan(1024, 64, 1 << 20, {'split_k': sk} if sk else None)['split_k'], ms=ms, gbs=4.0 * 2**30 / ms / 1e6)), flush=True)
ms = t_ms(lambda: shg.gen_omega(1 << 20, 64))
print(json.dumps(dict(gen_omega_2e20x64_ms=ms)))
res = {}
variants = [('auto', None), ('sk36', {'split_k': 36}), ('sk74', {'split_k': 74}), ('abox1', {'a_box': 1}),
            ('abox2_sk36', {'a_box': 2, 'split_k': 36})]
for rnd in range(3):
    for name, tune in variants:
        res.setdefault(name, []).append(t_ms(lambda: shg.shgemm(A, Om, tune=tune), reps=3))
for name, tune in variants:
    ms = sorted(res[name])[1]
    print(json.dumps(dict(mode='0-shgemm', variant=name, split_k=shg.plan(1024, 64, 1 << 20, tune)['split_k'], ms=ms, gbs=4.0 * 2**30 / ms / 1e6)), flush=True)
