"""Edge-shape fuzz (round 2): tiny and degenerate m, k, n (1..40 and a few larger), A and Omega as
padded slices of wider buffers (lda / ldo not equal to the extent, misaligned bases), both Omega
layouts, SHGEMM-FP16 / -TF32, K- and M-major A, random tunables; Y against the oracle bars.
Usage: python tools/fuzz_edge.py LO HI."""
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle as orc  # noqa: E402
orc.build()
import paper_2304_04612_b200 as shg  # noqa: E402
from gpu_common import check_bars, omega_bits, to_np  # noqa: E402


def pick(r):
    return int(r.choice([int(r.integers(1, 41)), int(r.integers(1, 41)), int(r.integers(41, 700)), 1, 2, 3, 4, 8]))


def run(i):
    r = np.random.default_rng(500000 + i)
    m, k, n = pick(r), pick(r), pick(r)
    kind = ["fp16", "fp16", "tf32"][i % 3]
    mmajor = bool(r.integers(0, 2))
    row_om = bool(r.integers(0, 2))
    pad_a, pad_o, off = int(r.integers(0, 5)), int(r.integers(0, 9)), int(r.integers(0, 3))
    tune = {}
    if r.random() < 0.3:
        tune["split_k"] = int(r.integers(1, 4))
    if r.random() < 0.2:
        tune["stream_k"] = int(r.integers(1, 3))
    A = (r.standard_normal((m, k)) * np.exp(r.uniform(-2, 2))).astype(np.float32)
    if mmajor:       # At (k x m) slice of a wider, offset buffer
        buf = torch.zeros(k * (m + pad_a) + off + 4, device="cuda")
        At = buf[off: off + k * (m + pad_a)].view(k, m + pad_a)[:, :m]
        At.copy_(torch.from_numpy(np.ascontiguousarray(A.T)).cuda())
    else:
        buf = torch.zeros(m * (k + pad_a) + off + 4, device="cuda")
        Ad = buf[off: off + m * (k + pad_a)].view(m, k + pad_a)[:, :k]
        Ad.copy_(torch.from_numpy(A).cuda())
    om_src = shg.gen_omega(k, n, seed=i, layout="row")
    if row_om:
        ob = torch.zeros(k * (n + pad_o) + off + 8, dtype=torch.float16, device="cuda")
        Om = ob[off: off + k * (n + pad_o)].view(k, n + pad_o)[:, :n]
    else:
        ob = torch.zeros(n * (k + pad_o) + off + 8, dtype=torch.float16, device="cuda")
        Om = ob[off: off + n * (k + pad_o)].view(n, k + pad_o)[:, :k].t()
    Om.copy_(om_src)
    try:
        Y = shg.shgemm_at(At, Om, tune=tune or None, tc=kind) if mmajor else shg.shgemm(Ad, Om, tune=tune or None,
                                                                                         tc=kind)
        torch.cuda.synchronize()
    except shg.SHGError as err:
        assert "INVALID" in str(err) and tune, err
        return
    ob_bits = omega_bits(om_src)
    if not np.any(orc.gemm_y64(A, ob_bits)):
        assert not np.any(to_np(Y)), "Y should be zero"
        return
    check_bars(orc, A, ob_bits, to_np(Y), ratio=2.0 if k >= 16 else float("inf"))


lo, hi = int(sys.argv[1]), int(sys.argv[2])
fails = 0
for i in range(lo, hi):
    try:
        run(i)
    except Exception as e:
        fails += 1
        print("FAIL", i, repr(e)[:300], flush=True)
        traceback.print_exc(limit=3)
print(f"fuzz_edge done: {hi - lo} cases, {fails} failures", flush=True)
