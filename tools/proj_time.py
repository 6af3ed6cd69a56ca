"""cfg3 (RP-HOSVD 1024^3, J = 64) projection timings: project() per mode (Omega generated in the
k-tiled layout + SHGEMM), and mode 0 split into generation and GEMM, k-tiled vs column-major Omega."""
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

T = shg.synth('gauss', 1, 0x102, 1024, 1024 * 1024).view(1024, 1024, 1024)


def t_ms(fn, reps=5):
    for _ in range(2):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


ws = torch.empty(max(shg.project_workspace_size([1024] * 3, md, 64) for md in range(3)), dtype=torch.uint8,
                 device='cuda')
for rnd in range(2):
    for mode in range(3):
        ms = t_ms(lambda: shg.project(T, mode, 64, workspace=ws))
        print(json.dumps(dict(round=rnd, mode=mode, project_ms=ms, gbs=4.0 * 2 ** 30 / ms / 1e6)), flush=True)
A = T.view(1024, -1)
K = 1 << 20
Om = shg.gen_omega(K, 64)
Omt = shg.gen_omega_tiled(K, 64)
Y = torch.empty(1024, 64, device='cuda')
sk_ws = torch.empty(max(1, shg.workspace_size(1024, 64, K)), dtype=torch.uint8, device='cuda')
for rnd in range(3):
    r = {"round": rnd,
         "gen_colmajor_ms": t_ms(lambda: shg.gen_omega(K, 64)),
         "gen_tiled_ms": t_ms(lambda: shg.gen_omega_tiled(K, 64)),
         "shgemm_colmajor_ms": t_ms(lambda: shg.shgemm(A, Om, out=Y, workspace=sk_ws)),
         "shgemm_tiled_ms": t_ms(lambda: shg.shgemm_tiled(A, Omt, 64, out=Y, workspace=sk_ws))}
    print(json.dumps(r), flush=True)
