"""TCEC-SGEMM (NEXT-2) timing: the pipelines' FP32 products on the tensor cores vs cuBLAS SGEMM
(TF32 off). Prints one JSON line per shape: ms, TFLOP/s (2mnk/t), algorithmic GB/s, plan."""
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


torch.backends.cuda.matmul.allow_tf32 = False
g = torch.Generator(device="cuda").manual_seed(0)
cases = [
    ("rsvd_line3 B^T = A^T Q (cfg2)", 16384, 272, 16384, True),
    ("hosvd_core step1 (cfg3)", 1 << 20, 64, 1024, True),
    ("hosvd_core step2 (cfg3)", 65536, 64, 1024, True),
    ("square 8192 x 8192 . 8192 x 256", 8192, 256, 8192, False),
    ("tall 1M x 4096 . 4096 x 128", 1 << 20, 128, 4096, False),
]
for name, m, n, k, mmajor in cases:
    X = torch.randn(k, m, device="cuda", generator=g) if mmajor else torch.randn(m, k, device="cuda", generator=g)
    A = X.t() if mmajor else X
    B = torch.randn(k, n, device="cuda", generator=g)
    C = torch.empty(m, n, device="cuda")
    ws = torch.empty(max(1, shg.tcec_workspace_size(m, n, k)), dtype=torch.uint8, device="cuda")
    t_tc = timeit(lambda: shg.tcec_sgemm(A, B, out=C, workspace=ws))
    t_sg = timeit(lambda: torch.matmul(A, B, out=C))
    flops = 2.0 * m * n * k
    byts = 4.0 * (m * k + k * n + m * n)
    print(json.dumps({"case": name, "m": m, "n": n, "k": k, "a_mn_major": mmajor,
                      "tcec_ms": t_tc, "tcec_tflops": flops / t_tc / 1e9, "tcec_gbs": byts / t_tc / 1e6,
                      "sgemm_ms": t_sg, "sgemm_tflops": flops / t_sg / 1e9, "speedup": t_sg / t_tc,
                      "plan": shg.tcec_plan(m, n, k)}), flush=True)
    del X, A, B, C, ws
    torch.cuda.empty_cache()
