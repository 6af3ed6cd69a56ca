"""Stream-K schedule (KParams::sk, shg_tune_t.stream_k): equal contiguous ranges of the
(tile, k-block) iterations per SM (pair), partial tiles summed in-kernel by the last piece in fixed k
order. Parity against the oracle bars on every mainloop variant, determinism, ragged shapes,
ranges shorter and longer than one tile, and concurrent stream-K kernels (no inter-CTA waiting, so
no co-residency is assumed)."""
import numpy as np
import pytest

from gpu_common import check_bars, omega_bits, to_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def shg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_04612_b200 import _build
    _build.build()
    import paper_2304_04612_b200 as m
    assert m.device_supported(), "device is not sm_100"
    return m


def _A(m, k, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(m, k, device="cuda", generator=g)


def test_stream_k_auto_rule(shg):
    """Auto: stream-K on the HBM side with a badly quantised last wave (m = k = 32768, n = 64..128:
    256 / 128 tiles on 148 / 74 units), whole tiles on the tensor side (no gain under the power cap)
    and where the waves are full."""
    assert shg.plan(32768, 128, 32768)["stream_k"] == 1
    assert shg.plan(32768, 64, 32768)["stream_k"] == 1
    assert shg.plan(32768, 256, 32768)["stream_k"] == 0
    assert shg.plan(16384, 272, 16384)["stream_k"] == 0
    assert shg.plan(1024, 64, 1 << 20)["stream_k"] == 0 and shg.plan(1024, 64, 1 << 20)["split_k"] > 1
    assert shg.plan(16384, 272, 16384, {"stream_k": 1})["stream_k"] == 1
    assert shg.plan(32768, 256, 32768, {"stream_k": 1})["stream_k"] == 1
    assert shg.plan(4194304, 256, 4096)["stream_k"] == 0
    assert shg.plan(512, 32, 512)["stream_k"] == 0 and shg.plan(512, 32, 512)["split_k"] == 1   # cfg1
    with pytest.raises(shg.SHGError):
        shg.plan(4096, 1024, 4096, {"stream_k": 1})              # several N tiles
    with pytest.raises(shg.SHGError):
        shg.plan(4096, 256, 4096, {"stream_k": 3})


@pytest.mark.parametrize("m,k,n,tune", [
    (2048, 4096, 256, {}),                    # pairs, 8 tiles on 74 units: ranges < one tile
    (20000, 3000, 256, {}),                   # 79 tiles: ranges ~ one tile, pieces straddle 2-3 tiles
    (40000, 1024, 128, {}),                   # 157 tiles, ranges > 2 tiles (full tiles in the middle)
    (5000, 5000, 272, {}),                    # wide tile (K_c = 64), ragged m
    (3000, 2000, 64, {}),                     # single CTAs, BN = 64
    (3000, 4000, 96, {"pair": 2}),
    (2500, 3000, 200, {"tc": "tf32"}),        # SHGEMM-TF32
    (700, 5000, 160, {"max_ctas": 40}),       # few units (grid cap)
])
def test_stream_k_bars_and_determinism(shg, orc, m, k, n, tune):
    A = _A(m, k, m + n)
    Om = shg.gen_omega(k, n, seed=5)
    t = dict(tune, stream_k=1)
    assert shg.plan(m, n, k, t)["stream_k"] == 1
    y1 = shg.shgemm(A, Om, tune=t)
    y2 = shg.shgemm(A, Om, tune=t)
    y0 = shg.shgemm(A, Om, tune=dict(tune, stream_k=2))
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)                                  # fixed-order fix-up
    rows = np.unique(np.linspace(0, m - 1, 300).astype(np.int64))
    A_h = to_np(A)
    check_bars(orc, A_h, omega_bits(Om), to_np(y1)[rows], rows=rows)
    # the same result up to summation order as whole tiles
    assert float((y1 - y0).abs().max()) <= 1e-4 * float(y0.abs().max())


def test_stream_k_mmajor_and_tcec(shg, orc):
    At = _A(3000, 9000, 1)                                       # A = At^T: m = 9000, k = 3000
    Om = shg.gen_omega(3000, 256, seed=2)
    y = shg.shgemm_at(At, Om, tune={"stream_k": 1})
    rows = np.arange(0, 9000, 37)
    check_bars(orc, np.ascontiguousarray(to_np(At).T[rows]), omega_bits(Om), to_np(y)[rows])
    B = _A(4096, 272, 3)
    A = _A(16384 // 4, 4096, 4)
    c1 = shg.tcec_sgemm(A, B, tune={"stream_k": 1})
    c0 = shg.tcec_sgemm(A, B, tune={"stream_k": 2})
    assert shg.tcec_plan(4096, 272, 4096, {"stream_k": 1})["stream_k"] == 1
    assert float((c1 - c0).abs().max()) <= 1e-5 * float(c0.abs().max())
    rr = np.arange(0, 4096, 41)
    Ah, Bh = to_np(A), to_np(B)
    e = orc.relative_error(to_np(c1)[rr], orc.gemm_y64_f32b(Ah[rr], Bh))
    assert e <= 1e-5


def test_stream_k_concurrent_kernels(shg):
    """Four stream-K projections on four streams at once: each kernel's grid is persistent, so
    they cannot all be resident; the last-arriving piece does the fix-up, nothing waits on another
    CTA, so they complete (bitwise equal to serial runs)."""
    A = _A(16384, 4096, 7)
    Om = shg.gen_omega(4096, 272, seed=1)
    ref = shg.shgemm(A, Om, tune={"stream_k": 1})
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = []
    for s in streams:
        with torch.cuda.stream(s):
            outs.append([shg.shgemm(A, Om, tune={"stream_k": 1}, stream=s) for _ in range(3)])
    torch.cuda.synchronize()
    for o in outs:
        for y in o:
            assert torch.equal(y, ref)


def test_stream_k_config2_full_size(shg, orc):
    """BASELINE config 2's projection (16384^2 . 16384 x 272) with stream-K (wide pair tile, 74
    units over 64 tiles), sampled rows against the oracle."""
    m = k = 16384
    n = 272
    A = shg.synth("gauss", 2, 0x101, m, k)
    Om = shg.gen_omega(k, n, seed=0)
    Y = shg.shgemm(A, Om, tune={"stream_k": 1})
    rows = np.unique(np.concatenate([np.arange(0, m, 97), [m - 1]]))
    A_s = orc.synth_rows("gauss", 2, 0x101, rows, k)
    check_bars(orc, A_s, omega_bits(Om), to_np(Y)[rows])


@pytest.mark.parametrize("variant", ["auto", "row_major", "tf32", "tcec_mmajor"])
def test_config2_projection_full_size_variants(shg, orc, variant):
    """BASELINE config 2's projection (16384^2 . 16384 x 272) on the default plan (one wide pair
    tile, staggered two-stage promotion), with §8(b)'s row-major Omega, on SHGEMM-TF32, and the
    pipeline's line-3 product B^T = A^T Q (TCEC-SGEMM, A read in place as MN-major, wide pair tile);
    sampled rows against the oracle."""
    m = k = 16384
    n = 272
    A = shg.synth("gauss", 3, 0x101, m, k)
    rows = np.unique(np.concatenate([np.arange(0, m, 131), [m - 1]]))
    if variant == "tcec_mmajor":
        Q = _A(k, n, 17)
        C = shg.tcec_sgemm(A.t(), Q)                     # (A^T) Q: A^T is MN-major, m x k = 16384^2
        At_rows = np.ascontiguousarray(to_np(A.t()[torch.from_numpy(rows).cuda()]))
        e = orc.relative_error(to_np(C)[rows], orc.gemm_y64_f32b(At_rows, to_np(Q)))
        assert e <= 1e-5, e
        return
    Om = shg.gen_omega(k, n, seed=0, layout="row" if variant == "row_major" else "col")
    Y = shg.shgemm(A, Om, tc="tf32" if variant == "tf32" else None)
    A_s = orc.synth_rows("gauss", 3, 0x101, rows, k)
    check_bars(orc, A_s, omega_bits(Om), to_np(Y)[rows])
