"""Small calls of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(600, 700, device="cuda", generator=g)
for n in (32, 130, 272):
    Om = shg.gen_omega(700, n, seed=1)
    shg.shgemm(A, Om)
    shg.shgemm(A, Om, tc="tf32")
    shg.shgemm(A, Om, tune={"split_k": 3})
    shg.tcec_sgemm(A, torch.randn(700, n, device="cuda", generator=g))
shg.shgemm_at(A, shg.gen_omega(600, 64, seed=2))          # A (600 x 700) read as the M-major At of a 700 x 600
T = torch.randn(40, 64, 96, device="cuda", generator=g)
for mode in range(3):
    shg.project(T, mode, 16)
shg.set_inkernel_omega(True)
shg.project(T, 0, 16)
shg.set_inkernel_omega(2)      # generator warps idle: every Omega tile from the stagers' fallback
shg.project(T, 0, 16)
shg.project(T, 1, 16)
shg.set_inkernel_omega(False)
# later paths: pairs, wide 288, k-tiled Omega, project slab views
# with S % 32 == 0 (second half of a stage continues in the next slab), row-sharded Omega, probes
A2 = torch.randn(1100, 512, device="cuda", generator=g)
Om2 = shg.gen_omega(512, 256, seed=3)
shg.shgemm(A2, Om2, tune={"pair": 1})
# round 2: row-major Omega (transpose pass; TF32 widening; CUDA-core fallback), stream-K (pairs, wide,
# single CTAs), several N tiles (evict_normal A), shgemm_host with a short last chunk
Om_row = shg.gen_omega(512, 256, seed=3, layout="row")
shg.shgemm(A2, Om_row)
shg.shgemm(A2, Om_row, tc="tf32")
shg.shgemm(A2, Om_row, tune={"force_simt": 1})
A3 = torch.randn(1100, 4096, device="cuda", generator=g)
for n, t in ((256, {"stream_k": 1}), (272, {"stream_k": 1}), (64, {"stream_k": 1, "pair": 2, "max_ctas": 64})):
    shg.shgemm(A3, shg.gen_omega(4096, n, seed=6), tune=t)
shg.shgemm(A2, shg.gen_omega(512, 600, seed=7))
shg.shgemm_host(A2.cpu().pin_memory(), Om_row, chunk_rows=512)
shg.shgemm(A2, shg.gen_omega(512, 288, seed=4))
shg.shgemm_tiled(A2, shg.gen_omega_tiled(512, 200, seed=5), 200)
T2 = torch.randn(6, 32, 96, device="cuda", generator=g)
shg.project(T2, 1, 24)
shg.project(T2, 1, 24, omega_row0=64, k_total=1024)
shg.probe_boxmuller(torch.arange(1 << 12, device="cuda", dtype=torch.int32) << 20)
torch.cuda.synchronize()
print("sanitize-small ok")
