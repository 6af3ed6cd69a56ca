"""Three TCEC-SGEMM calls at the RSVD line-3 shape (cfg2: B^T = A^T Q), for ncu captures."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(16384, 16384, device="cuda", generator=g)
Q = torch.randn(16384, 272, device="cuda", generator=g)
for _ in range(3):
    C = shg.tcec_sgemm(X.t(), Q)
torch.cuda.synchronize()
print("ok", float(C.abs().sum()))
