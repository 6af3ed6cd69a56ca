"""Round-2 fuzz of the other entry points: gen_omega (random k, n, seed, dist, stream_id, row0,
k_total, both layouts, padded ldo) bit-exact vs the oracle; tcec_sgemm with random A / B layouts and
padding vs the oracle's Eq-9 bars; shgemm_host with random chunk heights, padded host A / Y and
both Omega layouts vs the device shgemm. Usage: python tools/fuzz_misc.py LO HI."""
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle as orc  # noqa: E402
orc.build()
import paper_2304_04612_b200 as shg  # noqa: E402
from gpu_common import U32, omega_bits, to_np  # noqa: E402


def padded(rows, cols, pad, dtype, device, transpose=False):
    """(rows, cols) view with row pitch cols + pad (or the transpose of such a (cols, rows) view)."""
    if transpose:
        buf = torch.zeros(cols, rows + pad, dtype=dtype, device=device)
        return buf[:, :rows].t()
    buf = torch.zeros(rows, cols + pad, dtype=dtype, device=device)
    return buf[:, :cols]


def run(i):
    r = np.random.default_rng(700000 + i)
    kind = i % 3
    if kind == 0:     # Omega generator
        k, n = int(r.integers(1, 3000)), int(r.integers(1, 300))
        dist, sid, row0 = int(r.integers(0, 4)), int(r.integers(0, 5)), int(r.integers(0, 50))
        k_total = row0 + k + int(r.integers(0, 1000))
        layout = "row" if r.random() < 0.5 else "col"
        out = padded(k, n, int(r.integers(0, 9)), torch.float16, "cuda", transpose=(layout == "col"))
        shg.gen_omega(k, n, seed=i, dist=dist, stream_id=sid, row0=row0, k_total=k_total, out=out)
        ref = orc.omega_f16(k, n, seed=i, dist=dist, stream_id=sid, row0=row0, k_total=k_total)
        assert np.array_equal(omega_bits(out), ref), ("omega", k, n, dist, sid, row0, layout)
    elif kind == 1:   # TCEC-SGEMM
        m, k, n = int(r.integers(1, 900)), int(r.integers(1, 2000)), int(r.integers(1, 300))
        A = (r.standard_normal((m, k)) * np.exp(r.uniform(-3, 3))).astype(np.float32)
        B = (r.standard_normal((k, n)) * np.exp(r.uniform(-3, 3))).astype(np.float32)
        Ad = padded(m, k, int(r.integers(0, 5)), torch.float32, "cuda", transpose=bool(r.integers(0, 2)))
        Bd = padded(k, n, int(r.integers(0, 5)), torch.float32, "cuda", transpose=bool(r.integers(0, 2)))
        Ad.copy_(torch.from_numpy(A))
        Bd.copy_(torch.from_numpy(B))
        C = to_np(shg.tcec_sgemm(Ad, Bd)).astype(np.float64)
        y64 = orc.gemm_y64_f32b(A, B)
        Aa, Ba = np.abs(A).astype(np.float64), np.abs(B).astype(np.float64)
        bound = 1.2 * ((k / 8.0 + 9.0) * U32 * (Aa @ Ba) + 2.0 ** -35 * ((Aa < 2.0 ** -13) @ Ba + Aa @ (Ba < 2.0 ** -13)))
        assert np.all(np.abs(C - y64) <= bound + 1e-300), float(np.max(np.abs(C - y64) / np.maximum(bound, 1e-300)))
    else:             # host streaming
        m, k, n = int(r.integers(1, 3000)), int(r.integers(1, 2000)), int(r.integers(1, 300))
        layout = "row" if r.random() < 0.5 else "col"
        Om = shg.gen_omega(k, n, seed=i, layout=layout)
        A = torch.randn(m, k, generator=torch.Generator().manual_seed(i))
        A_h = padded(m, k, int(r.integers(0, 5)), torch.float32, "cpu")
        A_h.copy_(A)
        Y_h = padded(m, n, int(r.integers(0, 5)), torch.float32, "cpu")
        chunk = int(r.choice([0, 128, 256, 384, 1024]))
        shg.shgemm_host(A_h, Om, Y_h, chunk_rows=chunk)
        torch.cuda.synchronize()
        # per-chunk device products on the same rows: bitwise equal
        rows = shg.lib().shg_host_workspace_size(n, k, chunk, shg.OMEGA_ROW_MAJOR if layout == "row" else shg.OMEGA_COL_MAJOR)
        assert rows > 0
        # the device reference reads A with the same row pitch shgemm_host stages it at (k rounded
        # up to 4: the pitch decides between the tensor-core path and the CUDA-core fallback)
        Ad = padded(m, k, (k + 3) // 4 * 4 - k, torch.float32, "cuda")
        Ad.copy_(A)
        ch = chunk if chunk > 0 else None
        if ch is None:
            ref = shg.shgemm(Ad, Om)
            # the heuristic chunk may split m: compare within the bars instead of bitwise
            d = (Y_h.cuda() - ref).abs().max().item()
            assert d <= 1e-5 * max(1.0, ref.abs().max().item()), d
        else:
            ch = max(128, (ch + 127) // 128 * 128)
            ch = min(ch, (m + 127) // 128 * 128)
            ref = torch.cat([shg.shgemm(Ad[r0:r0 + ch], Om) for r0 in range(0, m, ch)])
            assert torch.equal(Y_h.cuda(), ref), "host streaming != device chunks"


lo, hi = int(sys.argv[1]), int(sys.argv[2])
fails = 0
for i in range(lo, hi):
    try:
        run(i)
    except Exception as e:
        fails += 1
        print("FAIL", i, repr(e)[:300], flush=True)
        traceback.print_exc(limit=3)
print(f"fuzz_misc done: {hi - lo} cases, {fails} failures", flush=True)
