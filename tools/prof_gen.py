"""Workload for ncu: the k-tiled Omega generator on cfg3's Omega (2^20 x 64), then project() on the
cfg3 tensor (mode 0) with in-kernel Omega and with the separate generator + SHGEMM."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_04612_b200 as shg  # noqa: E402

K = 1 << 20
T = shg.synth("gauss", 1, 0x102, 1024, 1024 * 1024).view(1024, 1024, 1024)
ws = torch.empty(shg.project_workspace_size([1024] * 3, 0, 64), dtype=torch.uint8, device="cuda")
W = torch.empty(1024, 64, device="cuda")
for _ in range(3):
    shg.gen_omega_tiled(K, 64)
    shg.project(T, 0, 64, workspace=ws, out=W)
torch.cuda.synchronize()
shg.gen_omega_tiled(K, 64)                       # launch: gen_omega_kernel
shg.set_inkernel_omega(True)
shg.project(T, 0, 64, workspace=ws, out=W)       # launch: shgemm_sm100_kernel<..., OMGEN>
shg.set_inkernel_omega(False)
shg.project(T, 0, 64, workspace=ws, out=W)       # launches: gen_omega_kernel, shgemm_sm100_kernel
torch.cuda.synchronize()
