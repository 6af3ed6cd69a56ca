"""RP-HOSVD cfg3 pipeline (noisy Alg-3 1024^3 tensor, ranks 64, TCEC core, CholeskyQR2) with every
Omega_(i) pre-generated on a side stream (pregen=True) vs generated inside each project() kernel
(pregen=False); interleaved rounds, median of 3 runs each; plus project() per mode both ways."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2304_04612_b200 as shg  # noqa: E402
from paper_2304_04612_b200 import pipelines as pl  # noqa: E402

T = synth.alg3_tensor_torch((1024, 1024, 1024), (64, 64, 64), pad=4, seed=1, noise=1e-2)
res = {}
for rnd in range(4):
    for pregen in (True, False):
        pl.rp_hosvd(T, (64, 64, 64), seed=0, timing=True, gemm="tcec", factor="gram", pregen=pregen)
        runs = [pl.rp_hosvd(T, (64, 64, 64), seed=0, timing=True, gemm="tcec", factor="gram", pregen=pregen)
                for _ in range(3)]
        r = sorted(runs, key=lambda x: x["times_ms"]["total"])[1]
        res.setdefault(pregen, []).append(r["times_ms"]["total"])
        if rnd == 0:
            print(json.dumps({"pregen": pregen, "lines_ms": r["times_ms"],
                              "residual": pl.hosvd_error(T, r["core"], r["Q"])}), flush=True)
for pregen, v in res.items():
    print(json.dumps({"pregen": pregen, "total_ms_median": statistics.median(v), "all": v}), flush=True)
