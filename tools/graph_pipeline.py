"""Experiment: RP-HOSVD (cfg3, product variant) captured once into a CUDA graph and replayed, vs the
eager pipeline: does removing host launch gaps between its ~40 kernels pay?"""
import json
import sys

import torch

sys.path.insert(0, '.')
import synth  # noqa: E402
from paper_2304_04612_b200 import pipelines as pl  # noqa: E402

T = synth.alg3_tensor_torch((1024, 1024, 1024), (64, 64, 64), pad=4, seed=1)
run = lambda: pl.rp_hosvd(T, (64, 64, 64), seed=0, gemm="tcec", factor="gram", check=False)  # noqa: E731


def t_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


eager = t_ms(run)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for _ in range(2):
        run()
torch.cuda.current_stream().wait_stream(side)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    out = run()
graph = t_ms(g.replay)
ref = run()
torch.cuda.synchronize()
same = bool(torch.allclose(out["core"], ref["core"], rtol=1e-5, atol=1e-6))
print(json.dumps({"pipeline": "rphosvd_cfg3", "eager_ms": eager, "graph_ms": graph, "graph_matches_eager": same,
                  "bad": int(out["bad"]) if out["bad"] is not None else None}), flush=True)
del T, g, out, ref
torch.cuda.empty_cache()
X = synth.spectrum_matrix_torch(synth.spectrum("exp", 16384, 256, 1e-2), seed=1)
run2 = lambda: pl.rsvd(X, 256, 16, seed=0, gemm="tcec", factor="gram", check=False)  # noqa: E731
eager2 = t_ms(run2)
try:
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            run2()
    torch.cuda.current_stream().wait_stream(side)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        out2 = run2()
    graph2 = t_ms(g2.replay)
    ok = True
except Exception as exc:  # noqa: BLE001
    graph2, ok = None, repr(exc)[:300]
print(json.dumps({"pipeline": "rsvd_cfg2", "eager_ms": eager2, "graph_ms": graph2, "captured": ok}))
