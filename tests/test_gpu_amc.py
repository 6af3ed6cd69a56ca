"""A multicast (shg_tune_t.a_mcast, shgemm_sm100_kernel<..., NPA>; DESIGN.md §5 "A read once"): a
cluster of NPA CTA pairs takes one m-block and NPA N tiles, and each A stage is fetched once per
cluster and multicast into the NPA CTAs that hold its rows (the loaded A count of PAPER.md:652,
mnk/b_n on the A100 design, becomes mk per cluster). The arithmetic is unchanged, so Y must be
BITWISE equal to the per-pair loads; plus the oracle bars on sampled rows, ragged m / k, both A
stage layouts, row-major Omega, padded A, several N groups per m-block, grid caps, and the
planner's eligibility rules."""
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


def test_a_mcast_plan_rules(shg):
    assert shg.plan(32768, 1024, 32768, {"a_mcast": 2})["a_mcast"] == 2
    assert shg.plan(32768, 1024, 32768, {"a_mcast": 4})["a_mcast"] == 4
    assert shg.plan(32768, 1024, 32768, {"a_mcast": 1})["a_mcast"] == 1
    assert shg.plan(32768, 768, 32768, {"a_mcast": 2, "bn": 192})["a_mcast"] == 2
    for bad in ({"a_mcast": 3}, {"a_mcast": 5}, {"a_mcast": -1},
                {"a_mcast": 4, "bn": 256, "split_k": 2},           # needs whole tiles
                {"a_mcast": 2, "pair": 2},                          # needs CTA pairs
                {"a_mcast": 2, "tc": "tf32"}):                      # SHGEMM-FP16 only
        with pytest.raises(shg.SHGError):
            shg.plan(32768, 1024, 32768, bad)
    with pytest.raises(shg.SHGError):
        shg.plan(32768, 768, 32768, {"a_mcast": 2})                 # 3 N tiles of 256
    with pytest.raises(shg.SHGError):
        shg.plan(32768, 256, 32768, {"a_mcast": 2})                 # one N tile
    with pytest.raises(shg.SHGError):
        shg.plan(16384, 272, 16384, {"a_mcast": 2})                 # wide tile


@pytest.mark.parametrize("m,k,n,tune", [
    (4096, 4096, 512, {"a_mcast": 2}),                       # one N group per m-block
    (4096, 4096, 1024, {"a_mcast": 4}),                      # clusters of 8 CTAs
    (4096, 4096, 1024, {"a_mcast": 2}),                      # two N groups per m-block
    (5000, 3000, 512, {"a_mcast": 2}),                       # ragged m (last pair half empty), k
    (1000, 2050, 384, {"a_mcast": 2, "bn": 192}),            # ragged k tail, BN 192
    (3000, 1000, 256, {"a_mcast": 2, "bn": 128}),            # BN 128, few k-blocks
    (6000, 4096, 512, {"a_mcast": 2, "a_box": 2}),           # 4-D row-pair A boxes
    (6000, 4096, 1024, {"a_mcast": 4, "max_ctas": 40}),      # grid cap: clusters loop over tiles
    (300, 640, 512, {"a_mcast": 2}),                         # fewer tiles than clusters
    (4096, 4096, 1000, {"a_mcast": 4}),                      # ragged n inside the last N tile
])
def test_a_mcast_bitwise_and_bars(shg, orc, m, k, n, tune):
    A = _A(m, k, m + n + k)
    Om = shg.gen_omega(k, n, seed=3)
    pl = shg.plan(m, n, k, tune)
    assert pl["a_mcast"] == tune["a_mcast"]
    off = dict(tune, a_mcast=1, split_k=1)      # the same whole-tile schedule without multicast
    y0 = shg.shgemm(A, Om, tune=off)
    y1 = shg.shgemm(A, Om, tune=tune)
    y2 = shg.shgemm(A, Om, tune=tune)
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.int32), y0.view(torch.int32))
    assert torch.equal(y1.view(torch.int32), y2.view(torch.int32))
    rows = np.unique(np.linspace(0, m - 1, 200).astype(np.int64))
    check_bars(orc, to_np(A), omega_bits(Om), to_np(y1)[rows], rows=rows)


def test_a_mcast_row_major_omega_and_padded_a(shg):
    """Row-major Omega (copied to the column-major operand) and an A with row padding (lda > k)."""
    m, k, n = 3000, 2000, 512
    A = _A(m, k + 40, 9)[:, :k]                                # lda = k + 40
    Om_rm = shg.gen_omega(k, n, seed=4, layout="row")
    y0 = shg.shgemm(A, Om_rm, tune={"a_mcast": 1, "split_k": 1})
    y1 = shg.shgemm(A, Om_rm, tune={"a_mcast": 2})
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.int32), y0.view(torch.int32))


def test_a_mcast_concurrent_streams(shg):
    """Clusters of 8 CTAs from four streams at once: cluster launches that do not fit wait for
    resources, nothing waits on another kernel (no co-residency assumed)."""
    m, k, n = 8192, 2048, 1024
    A = _A(m, k, 11)
    Om = shg.gen_omega(k, n, seed=6)
    ref = shg.shgemm(A, Om, tune={"a_mcast": 1, "split_k": 1})
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = []
    torch.cuda.synchronize()
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            outs.append(shg.shgemm(A, Om, tune={"a_mcast": 4 if i % 2 == 0 else 2}))
    torch.cuda.synchronize()
    for y in outs:
        assert torch.equal(y.view(torch.int32), ref.view(torch.int32))


def test_a_mcast_auto_rule_and_switch(shg):
    """Auto: 2 pairs per cluster whenever the N tiles pair up on the eligible path;
    shg_set_a_mcast overrides the default per process (explicit tunes win)."""
    assert shg.plan(32768, 1024, 32768)["a_mcast"] == 2
    assert shg.plan(32768, 512, 32768)["a_mcast"] == 2
    assert shg.plan(1 << 21, 512, 4096)["a_mcast"] == 2
    assert shg.plan(32768, 768, 32768)["a_mcast"] == 1           # 3 N tiles
    assert shg.plan(32768, 256, 32768)["a_mcast"] == 1           # one N tile
    assert shg.plan(16384, 272, 16384)["a_mcast"] == 1           # wide tile
    assert shg.plan(32768, 1024, 32768, {"tc": "tf32"})["a_mcast"] == 1
    assert shg.plan(32768, 1024, 32768, {"pair": 2})["a_mcast"] == 1
    assert shg.plan(4096, 512, 4096)["a_mcast"] == 1             # split-K plan (few tiles)
    prev = shg.set_a_mcast(1)
    try:
        assert shg.plan(32768, 1024, 32768)["a_mcast"] == 1
        assert shg.plan(32768, 1024, 32768, {"a_mcast": 2})["a_mcast"] == 2
        shg.set_a_mcast(4)
        assert shg.plan(32768, 1024, 32768)["a_mcast"] == 4
        assert shg.plan(32768, 768, 32768)["a_mcast"] == 1      # not eligible: silently off
    finally:
        shg.set_a_mcast(prev)
    with pytest.raises(ValueError):
        shg.set_a_mcast(3)


@pytest.mark.parametrize("dims,mode", [((9600, 32, 64), 0), ((48, 9600, 64), 1), ((96, 9600, 32), 1)])
def test_a_mcast_project_unfoldings(shg, dims, mode):
    """project() with n = 512 (2 N tiles, >= 74 pair tiles: whole tiles, auto A multicast) on K-major
    unfolding views, incl. the 3-D middle-mode view whose 64-k stage wraps into the next slab
    (S = 32): bitwise equal with the multicast switched off."""
    g = torch.Generator(device="cuda").manual_seed(sum(dims) + mode)
    T = torch.randn(*dims, device="cuda", generator=g)
    n = 512
    M = dims[mode]
    assert shg.plan(M, n, T.numel() // M)["a_mcast"] == 2
    y1 = shg.project(T, mode, n, seed=7)
    prev = shg.set_a_mcast(1)
    try:
        y0 = shg.project(T, mode, n, seed=7)
    finally:
        shg.set_a_mcast(prev)
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.int32), y0.view(torch.int32))


def test_a_mcast_not_on_mmajor(shg, orc):
    """shgemm_at (M-major A) keeps per-pair loads; results meet the bars with n = 512."""
    m, k, n = 3000, 2048, 512
    At = _A(k, m, 21)                     # A = At^T, M-major
    Om = shg.gen_omega(k, n, seed=2)
    y = shg.shgemm_at(At, Om)
    torch.cuda.synchronize()
    rows = np.unique(np.linspace(0, m - 1, 100).astype(np.int64))
    check_bars(orc, to_np(At).T.copy(), omega_bits(Om), to_np(y)[rows], rows=rows)
