"""Fig 6 analogue on B200: TFLOP/s (2mnk/t) of SHGEMM-FP16 / -TF32 and TCEC-SGEMM
(this library) vs cuBLAS SGEMM and cuBLAS TF32 GEMM, square sizes and the tall-skinny products of a
rank-512 randomized SVD of an m x m matrix (m x m . m x 512). Median of 5 timed calls after warm-up."""
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402


def t_ms(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return sorted(ts)[len(ts) // 2]


def case(kind, m, n, k):
    A = shg.synth("gauss", 7, 0x201, m, k)
    Om = shg.gen_omega(k, n, seed=1)
    B32 = Om.float()
    Y = torch.empty(m, n, device="cuda")
    fl = 2.0 * m * n * k
    r = {"kind": kind, "m": m, "n": n, "k": k}
    r["shgemm_fp16"] = fl / t_ms(lambda: shg.shgemm(A, Om, out=Y)) / 1e9
    r["shgemm_tf32"] = fl / t_ms(lambda: shg.shgemm(A, Om, out=Y, tc="tf32")) / 1e9
    r["tcec_fp16"] = fl / t_ms(lambda: shg.tcec_sgemm(A, B32, out=Y)) / 1e9
    torch.backends.cuda.matmul.allow_tf32 = False
    r["cublas_sgemm"] = fl / t_ms(lambda: torch.matmul(A, B32, out=Y)) / 1e9
    torch.backends.cuda.matmul.allow_tf32 = True
    r["cublas_tf32"] = fl / t_ms(lambda: torch.matmul(A, B32, out=Y)) / 1e9
    torch.backends.cuda.matmul.allow_tf32 = False
    print(json.dumps(r), flush=True)
    del A, Om, B32, Y
    torch.cuda.empty_cache()


for N in (1024, 2048, 4096, 8192, 16384):
    case("square", N, N, N)
for m in (4096, 8192, 16384, 32768, 65536):
    case("rsvd_rank512", m, 512, m)
