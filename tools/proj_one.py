"""Three project() calls (cfg3 mode 0: 1024^3 tensor, n = 64, k-tiled Omega) for ncu captures."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

T = shg.synth('gauss', 1, 0x102, 1024, 1024 * 1024).view(1024, 1024, 1024)
for _ in range(3):
    W = shg.project(T, 0, 64)
torch.cuda.synchronize()
print("ok", float(W.abs().sum()))
