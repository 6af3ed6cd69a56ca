"""Fig 5 analogue on B200: relative Frobenius error vs FP64 of A_F32 . B_F16 for
A ~ U(0,1) or N(0,1) and B ~ N(0,1) (FP16, from gen_omega), m = n = k: SHGEMM-FP16 and -TF32 (this
library), TCEC-SGEMM (this library, B widened to FP32), cuBLAS SGEMM (TF32 off) and cuBLAS TF32."""
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402


def rel(C, C64):
    return float(torch.linalg.norm(C.double() - C64) / torch.linalg.norm(C64))


for dist in ("uniform", "gauss"):
    for N in (256, 512, 1024, 2048, 4096, 8192, 16384):
        A = shg.synth("uniform" if dist == "uniform" else "gauss", 7, 0x200, N, N)
        Om = shg.gen_omega(N, N, seed=3)              # column-major FP16 view
        B32 = Om.float()
        C64 = A.double() @ B32.double()
        r = {"dist_A": dist, "m=n=k": N}
        r["shgemm_fp16"] = rel(shg.shgemm(A, Om), C64)
        r["shgemm_tf32"] = rel(shg.shgemm(A, Om, tc="tf32"), C64)
        r["tcec_fp16"] = rel(shg.tcec_sgemm(A, B32), C64)
        torch.backends.cuda.matmul.allow_tf32 = False
        r["cublas_sgemm"] = rel(A @ B32, C64)
        torch.backends.cuda.matmul.allow_tf32 = True
        r["cublas_tf32"] = rel(A @ B32, C64)
        torch.backends.cuda.matmul.allow_tf32 = False
        print(json.dumps(r), flush=True)
        del A, Om, B32, C64
        torch.cuda.empty_cache()
