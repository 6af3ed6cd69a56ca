"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs. Bars: Omega and the split bit-exact; Y within the north_star bars;
exact-arithmetic cases bit-exact."""
import json
import os

import numpy as np
import pytest

import synth
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


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ------------------------------------------------------------------------------------------ Omega
@pytest.mark.parametrize("k,n,seed,dist,stream_id,row0", [
    (512, 32, 0, 0, 0, 0),             # config 1
    (16384, 272, 0, 0, 0, 0),          # config 2 (4.46M elements)
    (1001, 17, 123, 0, 5, 3),          # ragged, odd row offset
    (4096, 256, 0, 0, 0, 0),           # config 4
    (3000, 40, 9, 1, 2, 0),            # Rademacher
    (3000, 40, 9, 2, 2, 8),            # s = 3
    (10000, 33, 9, 3, 1, 0),           # very sparse s = sqrt(k)
])
def test_omega_bit_exact(shg, orc, k, n, seed, dist, stream_id, row0):
    Om = shg.gen_omega(k, n, seed=seed, dist=dist, stream_id=stream_id, row0=row0)
    torch.cuda.synchronize()
    ref = orc.omega_f16(k, n, seed=seed, dist=dist, stream_id=stream_id, row0=row0, k_total=k)
    got = omega_bits(Om)
    assert got.shape == ref.shape
    mism = int(np.sum(got != ref))
    assert mism == 0, f"{mism} mismatches"


def test_omega_bit_exact_1e8(shg, orc):
    """>= 1e8 elements at the config-3 shape (K = 2^20 rows, n = 64 per mode, stream = mode)."""
    total = 0
    for mode in range(2):
        Om = shg.gen_omega(1 << 20, 64, seed=0, stream_id=mode)
        ref = orc.omega_f16(1 << 20, 64, seed=0, stream_id=mode)
        assert np.array_equal(omega_bits(Om), ref)
        total += ref.size
    assert total >= 1e8


# ------------------------------------------------------------------------------------------ split
def test_boxmuller_steps_exhaustive(shg, orc):
    """The generator's radius and cos/sin (OMEGA_SPEC §3.1-3.2; Gaussian Omega) on
    every one of the 2^24 codes, bit for bit against the oracle's fixed-operation versions; random
    low 8 bits (ignored by both) on a second pass."""
    code = np.arange(1 << 24, dtype=np.uint32)
    for low in (0, None):
        w = code << np.uint32(8)
        if low is None:
            w = w | np.random.default_rng(3).integers(0, 256, code.size).astype(np.uint32)
        r, c, s = shg.probe_boxmuller(torch.from_numpy(w.view(np.int32)).cuda())
        torch.cuda.synchronize()
        np.testing.assert_array_equal(r.cpu().numpy().view(np.uint32), orc.radius_spec_batch(w).view(np.uint32))
        oc, os_ = orc.sincos_spec_batch(w)
        np.testing.assert_array_equal(c.cpu().numpy().view(np.uint32), oc.view(np.uint32))
        np.testing.assert_array_equal(s.cpu().numpy().view(np.uint32), os_.view(np.uint32))


def test_split_exhaustive_all_fp32(shg, orc):
    """Device split (the mainloop's device function) == oracle split on all 2^32 FP32 patterns."""
    chunk = 1 << 28
    for c in range((1 << 32) // chunk):
        lo_pat = c * chunk
        bits = torch.arange(lo_pat, lo_pat + chunk, dtype=torch.int64, device="cuda").to(torch.int32)
        a = bits.view(torch.float32)
        hi, lo = shg.split(a)
        hi_np = to_np(hi).view(np.uint16)
        lo_np = to_np(lo).view(np.uint16)
        a_np = np.arange(lo_pat, lo_pat + chunk, dtype=np.uint64).astype(np.uint32).view(np.float32)
        rhi, rlo = orc.split(a_np)
        nan = np.isnan(a_np)
        ok_hi = (hi_np == rhi) | (nan & ((hi_np & 0x7C00) == 0x7C00) & ((hi_np & 0x3FF) != 0))
        # lo of NaN / inf inputs: NaN class compare
        lo_nan_g = ((lo_np & 0x7C00) == 0x7C00) & ((lo_np & 0x3FF) != 0)
        lo_nan_r = ((rlo & 0x7C00) == 0x7C00) & ((rlo & 0x3FF) != 0)
        ok_lo = (lo_np == rlo) | (lo_nan_g & lo_nan_r)
        assert ok_hi.all(), hex(int(a_np.view(np.uint32)[~ok_hi][0]))
        assert ok_lo.all(), hex(int(a_np.view(np.uint32)[~ok_lo][0]))


# ------------------------------------------------------------------------------------------ probes
def _probe_inputs(n=64):
    A = np.zeros((128, 64), np.float16)
    B = np.zeros((n, 64), np.float16)
    return A, B


def test_probe_umma_exact_small_integers(shg):
    """128 x 64 x 64 MMA on small integers is exact: validates descriptors, swizzle, TMEM ld."""
    rng = np.random.default_rng(0)
    A = rng.integers(-4, 5, size=(128, 64)).astype(np.float16)
    B = rng.integers(-4, 5, size=(64, 64)).astype(np.float16)
    D = shg.probe_umma(cuda(A.view(np.int16)), cuda(B.view(np.int16)), None, mode=0, nsteps=4)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    assert np.array_equal(to_np(D).astype(np.float64), ref)
    D1 = shg.probe_umma(cuda(A.view(np.int16)), cuda(B.view(np.int16)), None, mode=0, nsteps=1)
    ref1 = A[:, :16].astype(np.float64) @ B[:, :16].astype(np.float64).T
    assert np.array_equal(to_np(D1).astype(np.float64), ref1)


def test_probe_scale_input_d(shg):
    """The fold the mainloop relies on: first MMA with scale-input-d = 11 computes
    D = D_init * 2^-11 + A_0 B_0^T (then the rest accumulate)."""
    rng = np.random.default_rng(1)
    A = rng.integers(-3, 4, size=(128, 64)).astype(np.float16)
    B = rng.integers(-3, 4, size=(32, 64)).astype(np.float16)
    Dinit = (rng.integers(-2048 * 8, 2048 * 8, size=(128, 32))).astype(np.float32)
    D = shg.probe_umma(cuda(A.view(np.int16)), cuda(B.view(np.int16)), cuda(Dinit), mode=1, nsteps=4)
    ref = Dinit.astype(np.float64) * 2.0 ** -11 + A.astype(np.float64) @ B.astype(np.float64).T
    assert np.array_equal(to_np(D).astype(np.float64), ref)


def test_probe_accumulation_semantics(shg):
    """Record B200 tensor-core accumulation behaviour (PAPER.md:505-512 lists A100's):
    D = 1 plus one product 1.5 * 2^-24 -> RN gives 1 + 2^-23, RZ gives 1. Results go to
    gpurun_out/probe_semantics.json; the mainloop's correctness does not depend on them."""
    res = {}
    for name, a, b, d0 in [("pos_1.5ulp_half", 1.5 * 2 ** -12, 2 ** -12, 1.0),
                           ("neg_1.5ulp_half", -1.5 * 2 ** -12, 2 ** -12, -1.0),
                           ("pos_0.75ulp", 0.75 * 2 ** -12, 2 ** -12, 1.0),
                           ("pos_tiny_2^-30", 2 ** -15, 2 ** -15, 1.0)]:
        A, B = _probe_inputs(16)
        A[:, 0] = a
        B[:, 0] = b
        Dinit = np.full((128, 16), d0, np.float32)
        D = to_np(shg.probe_umma(cuda(A.view(np.int16)), cuda(B.view(np.int16)), cuda(Dinit), mode=0, nsteps=1))
        res[name] = float(D[0, 0]) - d0
    # many small terms inside one K=16 instruction: 16 x 2^-25 on top of 1.0
    A, B = _probe_inputs(16)
    A[:, :16] = 2 ** -13
    B[:, :16] = 2 ** -12
    D = to_np(shg.probe_umma(cuda(A.view(np.int16)), cuda(B.view(np.int16)), cuda(np.ones((128, 16), np.float32)),
                             mode=0, nsteps=1))
    res["16x2^-25_on_1"] = float(D[0, 0]) - 1.0
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "probe_semantics.json"), "w") as f:
        json.dump(res, f, indent=1)
    # DESIGN R4, the premise of the per-chunk RN promotion (P:505-512 found the same on A100):
    # 1 + 0.75 ulp(1) stays 1 (RN would give 1 + 2^-23), and -1 - 0.75 ulp stays -1 (RD would give
    # -(1 + 2^-23)): the accumulator add truncates toward zero (RZ)
    assert res["pos_1.5ulp_half"] == 0.0, res
    assert res["neg_1.5ulp_half"] == 0.0, res
    assert res["pos_0.75ulp"] == 0.0 and res["pos_tiny_2^-30"] == 0.0, res
    # ... while 16 products of 2^-25 inside one K = 16 instruction are summed exactly before the
    # accumulator add (1 + 2^-21 exactly): the products of one instruction are fused with extra bits
    assert res["16x2^-25_on_1"] == 2.0 ** -21, res


# ------------------------------------------------------------------------------------------ SHGEMM
def _run(shg, A, k, n, seed=0, dist=0, tune=None):
    Om = shg.gen_omega(k, n, seed=seed, dist=dist)
    Y = shg.shgemm(cuda(A), Om, tune=tune)
    torch.cuda.synchronize()
    return omega_bits(Om), to_np(Y)


def test_identity_omega_reconstructs_split(shg, orc):
    """Omega = [I; 0]: Y[i][j] = hi + lo 2^-11 of A[i][j] exactly (22-bit sum fits FP32)."""
    m, k, n = 256, 192, 128
    A = synth.gaussian(m, k, seed=3) * np.float32(7.0)
    eye = np.eye(k, n, dtype=np.float32).astype(np.float16)
    Om = torch.from_numpy(np.ascontiguousarray(eye.T)).cuda().t()      # column-major (k, n)
    Y = to_np(shg.shgemm(cuda(A), Om))
    hi, lo = orc.split(A[:, :n])
    rec = (hi.view(np.float16).astype(np.float64) + lo.view(np.float16).astype(np.float64) * 2.0 ** -11)
    rec = rec.reshape(m, n).astype(np.float32)
    assert np.array_equal(Y, rec)
    frac = np.mean(Y != A[:, :n])
    assert 0.15 < frac < 0.35


def test_exact_integer_case_bitwise(shg, orc):
    """Small-integer A with Rademacher Omega: exact arithmetic -> Y_gpu == exact product."""
    m, k, n = 300, 2048, 64
    A = synth.small_int_matrix(m, k, seed=5)
    om, Y = _run(shg, A, k, n, seed=3, dist=1)
    assert np.array_equal(Y.astype(np.float64), orc.gemm_y64(A, om))


def test_fp16_exact_A_split_is_exact(shg, orc):
    """A exactly FP16-representable: lo == 0 and Y == sum of hi products (north_star)."""
    m, k, n = 200, 512, 48
    A = synth.gaussian(m, k, seed=9).astype(np.float16).astype(np.float32)
    om, Y = _run(shg, A, k, n, seed=1)
    check_bars(orc, A, om, Y)


CASES = [
    # (m, k, n, dist_A)        -- several tiles, ragged tails in every dimension
    (512, 512, 32, "spectrum"),    # BASELINE config 1
    (512, 512, 32, "normal"),
    (512, 512, 32, "uniform"),
    (300, 1000, 50, "normal"),
    (129, 65, 17, "normal"),
    (1000, 777, 272, "normal"),    # two N tiles of 144
    (640, 4096, 256, "normal"),
    (256, 3000, 512, "uniform"),   # two N tiles of 256
    (130, 64, 16, "normal"),
    (384, 16384, 64, "normal"),    # split-K
]


@pytest.mark.parametrize("m,k,n,kind", CASES)
def test_shgemm_bars(shg, orc, m, k, n, kind):
    if kind == "spectrum":
        A = synth.spectrum_matrix(synth.spectrum("exp", m, 22, 1e-2), seed=1)[:, :k]
    elif kind == "normal":
        A = synth.gaussian(m, k, seed=m + k)
    else:
        A = synth.uniform(m, k, seed=m + k)
    om, Y = _run(shg, A, k, n)
    check_bars(orc, A, om, Y)


@pytest.mark.parametrize("tune", [{"force_simt": 1}, {"split_k": 3}, {"bn": 64}, {"max_ctas": 3}, {"pair": 1},
                                  {"pair": 2}, {"pair": 1, "bn": 144}, {"pair": 1, "split_k": 2, "max_ctas": 6},
                                  {"a_box": 1}, {"a_box": 1, "pair": 1}, {"a_box": 1, "split_k": 4}])
def test_shgemm_tunables(shg, orc, tune):
    m, k, n = 400, 1500, 100
    A = synth.gaussian(m, k, seed=2)
    om, Y = _run(shg, A, k, n, tune=tune)
    check_bars(orc, A, om, Y)


def test_deterministic(shg):
    A = cuda(synth.gaussian(700, 3000, seed=4))
    Om = shg.gen_omega(3000, 200, seed=1)
    Y1 = shg.shgemm(A, Om).clone()
    Y2 = shg.shgemm(A, Om)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)


def test_misaligned_leading_dims_fall_back(shg, orc):
    m, k, n = 100, 130, 20
    Afull = synth.gaussian(m, k + 3, seed=8)
    A = cuda(Afull)[:, 1:k + 1]              # lda = k + 3 (not % 4), base offset 4 B
    Om = shg.gen_omega(k, n, seed=2)
    Y = to_np(shg.shgemm(A, Om))
    check_bars(orc, Afull[:, 1:k + 1], omega_bits(Om), Y)


def test_edge_sizes(shg):
    Om = shg.gen_omega(0, 5)
    Y = shg.shgemm(torch.zeros((3, 0), device="cuda"), Om)
    torch.cuda.synchronize()
    assert torch.equal(Y, torch.zeros((3, 5), device="cuda"))
    Y = shg.shgemm(torch.zeros((0, 8), device="cuda"), shg.gen_omega(8, 4))
    assert Y.shape == (0, 4)


def test_fp16_range_failure_is_flagged(shg):
    """|a| > 65504 -> non-finite Y rows and the flag (PAPER.md:705-706 'expected to fail')."""
    A = synth.cauchy_like(256, seed=0)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    Om = shg.gen_omega(256, 32, seed=0)
    Y = to_np(shg.shgemm(cuda(A), Om, nonfinite=flag))
    assert int(flag.item()) == 1
    bad_rows = np.any(np.abs(A) >= 65520, axis=1)
    assert bad_rows.any()
    assert np.all(np.any(~np.isfinite(Y[bad_rows]), axis=1))
    assert np.all(np.isfinite(Y[~bad_rows]))


# ------------------------------------------------------------------------------------------ synth / full size
def test_device_synth_matches_oracle_rows(shg, orc):
    A = shg.synth("gauss", 2, 0x100, 300, 1000, row0=77)
    rows = np.array([0, 1, 150, 299]) + 77
    ref = orc.synth_rows("gauss", 2, 0x100, rows, 1000)
    assert np.array_equal(to_np(A)[rows - 77], ref)
    U = shg.synth("unif", 5, 0x101, 10, 64)
    assert np.array_equal(to_np(U), orc.synth_rows("unif", 5, 0x101, np.arange(10), 64))


def test_config4_full_size_sampled(shg, orc):
    """BASELINE config 4 at full size (A 4,194,304 x 4096 FP32 = 64 GiB on the device), the
    launch configuration bench.py times; 256 sampled rows (first/last + random) checked."""
    m, k, n = 4194304, 4096, 256
    free, _ = torch.cuda.mem_get_info()
    if free < (m * k * 4 + m * n * 4) * 1.05:
        pytest.skip("not enough device memory")
    A = shg.synth("gauss", 2, 0x100, m, k)
    Om = shg.gen_omega(k, n, seed=0)
    Y = shg.shgemm(A, Om)
    # the same product through §8(b)'s row-major Omega: bitwise the same Y at full size
    Y_rm = shg.shgemm(A[: 1 << 20], shg.gen_omega(k, n, seed=0, layout="row"))
    assert torch.equal(Y_rm, Y[: 1 << 20])
    del Y_rm
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([[0, 127, 128, m - 1], rng.integers(0, m, 252)]))
    Arows = orc.synth_rows("gauss", 2, 0x100, rows, k)
    assert np.array_equal(to_np(A[torch.from_numpy(rows).cuda()]), Arows)
    Ys = to_np(Y[torch.from_numpy(rows).cuda()])
    del A, Y
    torch.cuda.empty_cache()
    check_bars(orc, Arows, omega_bits(Om), Ys)


@pytest.mark.parametrize("variant", ["fp16", "split_k", "tf32", "mmajor"])
def test_int64_indexing_large_m(shg, orc, variant):
    """m * ldc > 2^31 (12.6M rows x 256 columns of Y) and m * k > 2^31 elements of A: the epilogue's
    row * ldc, the TMA row coordinates and the synthetic generator's offsets stay 64-bit; rows past
    2^31 / n and the last tile (ragged) checked against the oracle."""
    m, k, n = 12_600_001 if variant != "mmajor" else 12_600_004, 192, 256    # M-major: lda % 4 == 0
    Om = shg.gen_omega(k, n, seed=7)
    if variant == "mmajor":           # A stored k x m (M-major), rows of the product = columns of At
        At = shg.synth("gauss", 7, 0x107, k, m)
        Y = shg.shgemm_at(At, Om)
        A = At.t()
    else:
        A = shg.synth("gauss", 7, 0x107, m, k)
        Y = shg.shgemm(A, Om, tune={"split_k": 2} if variant == "split_k" else None,
                       tc="tf32" if variant == "tf32" else "fp16")
    torch.cuda.synchronize()
    rows = np.array([0, 1, (1 << 31) // n - 1, (1 << 31) // n, (1 << 31) // n + 1, 11_000_000, m - 257,
                     m - 2, m - 1])
    ridx = torch.from_numpy(rows).cuda()
    Arows = to_np(A[ridx])
    if variant != "mmajor":
        assert np.array_equal(Arows, orc.synth_rows("gauss", 7, 0x107, rows, k))
    Ys = to_np(Y[ridx])
    del A, Y
    torch.cuda.empty_cache()
    check_bars(orc, Arows, omega_bits(Om), Ys)


def test_project_tensor_over_2g_elements(shg, orc):
    """A 2100 x 1024 x 1024 tensor (2.25e9 elements > 2^31, 9 GB): every unfolding's projection with
    n = 16 (mode 0 K-major, mode 1 slab view, mode 2 M-major in place), sampled rows vs the oracle."""
    dims = (2100, 1024, 1024)
    T = shg.synth("gauss", 8, 0x108, dims[0], dims[1] * dims[2]).view(*dims)
    for mode in range(3):
        I = dims[mode]
        rows = np.array([0, 1, I // 2, I - 2, I - 1])
        ridx = torch.from_numpy(rows).cuda()
        W = shg.project(T, mode, 16, seed=8)
        U = to_np(torch.movedim(T, mode, 0)[ridx].reshape(len(rows), -1))
        ob = orc.omega_f16(U.shape[1], 16, seed=8, stream_id=mode)
        check_bars(orc, U, ob, to_np(W[ridx]))


def test_concurrent_streams_and_threads(shg):
    """Eight host threads, each on its own CUDA stream, issue shgemm / project / tcec_sgemm calls
    with library-allocated split-K workspaces concurrently: results bitwise equal to serial calls
    (the library keeps no shared mutable state but the launch counter and the per-device occupancy
    cache)."""
    import threading
    g = torch.Generator(device="cuda").manual_seed(21)
    A = torch.randn(700, 3000, device="cuda", generator=g)
    B = torch.randn(3000, 100, device="cuda", generator=g)
    T = torch.randn(20, 30, 40, device="cuda", generator=g)
    Om = shg.gen_omega(3000, 100, seed=2)
    calls = [lambda s: shg.shgemm(A, Om, stream=s), lambda s: shg.shgemm(A, Om, tune={"split_k": 5}, stream=s),
             lambda s: shg.project(T, 1, 12, seed=4, stream=s), lambda s: shg.tcec_sgemm(A, B, stream=s)]
    ref = [c(None) for c in calls]
    torch.cuda.synchronize()
    out = [[None] * len(calls) for _ in range(8)]
    err = []

    def worker(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    for i, c in enumerate(calls):
                        out[t][i] = c(s)
            s.synchronize()
        except Exception as e:        # surfaced below
            err.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not err, err
    for t in range(8):
        for i in range(len(calls)):
            assert torch.equal(out[t][i], ref[i]), (t, i)


def test_config5_full_size_sampled(shg, orc):
    """BASELINE config 5 at full size (A 32768^2 FP32 = 4 GiB) for n = 16 and 128 (HBM-bound,
    stream-K plans; n = 128 with the row-major Omega of §8(b)), n = 1024 and n = 4096 (tensor-bound,
    several N tiles): 64 sampled rows each against the oracle."""
    m = k = 32768
    A = shg.synth("gauss", 5, 0x105, m, k)
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([[0, 255, 256, m - 1], rng.integers(0, m, 60)]))
    ridx = torch.from_numpy(rows).cuda()
    Arows = to_np(A[ridx])
    assert np.array_equal(Arows[:3], orc.synth_rows("gauss", 5, 0x105, rows[:3], k))
    for n in (16, 128, 1024, 4096):       # 16 / 128: stream-K plans (auto), 1024 / 4096: 4 / 16 N tiles
        Om = shg.gen_omega(k, n, seed=n, layout="row" if n == 128 else "col")
        Ys = to_np(shg.shgemm(A, Om)[ridx])
        check_bars(orc, Arows, omega_bits(Om), Ys)
        del Om


def test_config3_project_full_size_sampled(shg, orc):
    """BASELINE config 3's projections at full size: a 1024^3 FP32 tensor (4 GiB), W = A_(i) Omega_(i)
    with n = 64 and K = 2^20 for every mode (mode 0 K-major, mode 1 a 3-D slab view, mode 2 M-major in
    place), in bench.py's launch configuration; 16 sampled rows of each W against the oracle with the
    oracle's own Omega_(i) (stream_id = mode). project()'s default generates Omega_(i) inside the
    projection kernel; the same call with the separate generator gives W bit for bit."""
    I = 1024
    T = shg.synth("gauss", 3, 0x103, I, I * I).view(I, I, I)
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([[0, 127, 128, I - 1], rng.integers(0, I, 12)]))
    ridx = torch.from_numpy(rows).cuda()
    prev = shg.get_inkernel_omega()
    for mode in range(3):
        shg.set_inkernel_omega(True)
        W = shg.project(T, mode, 64, seed=0)
        shg.set_inkernel_omega(False)
        W_sep = shg.project(T, mode, 64, seed=0)
        shg.set_inkernel_omega(prev)
        assert torch.equal(W, W_sep)
        U = to_np(torch.movedim(T, mode, 0)[ridx].reshape(len(rows), -1))
        ob = orc.omega_f16(I * I, 64, seed=0, stream_id=mode)
        check_bars(orc, U, ob, to_np(W[ridx]))


# ------------------------------------------------------------------------------------------ project
@pytest.mark.parametrize("dims", [(24, 40, 64), (16, 128, 32), (10, 12, 14)])
def test_project_all_modes(shg, orc, dims):
    from oracle import pipelines as pl
    T = synth.gaussian(int(np.prod(dims)), 1, seed=sum(dims)).reshape(dims)
    Tt = cuda(T)
    for mode in range(3):
        n = 24
        W = to_np(shg.project(Tt, mode, n, seed=3))
        U = np.ascontiguousarray(pl.unfold(T, mode))
        om = orc.omega_f16(U.shape[1], n, seed=3, stream_id=mode)
        check_bars(orc, U, om, W)


# ------------------------------------------------------------------------------------------ M-major A
@pytest.mark.parametrize("m,k,n,tune", [(300, 1000, 50, None), (128, 4096, 256, None), (1000, 777, 272, None),
                                        (77, 3000, 64, {"split_k": 5}), (200, 300, 40, {"force_simt": 1})])
def test_shgemm_at_mmajor(shg, orc, m, k, n, tune):
    """A given M-major (At = A^T row-major): the last-mode unfolding path of project()."""
    A = synth.gaussian(m, k, seed=m + 3 * k)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    Om = shg.gen_omega(k, n, seed=6)
    Y = to_np(shg.shgemm_at(At, Om, tune=tune))
    check_bars(orc, A, omega_bits(Om), Y)


def test_project_fast_paths_large(shg, orc):
    """Modes 0 (K-major), 1 (3-D K-major view, S = 256) and 2 (M-major, in place) on a tensor big
    enough for the tensor-core path with split-K."""
    from oracle import pipelines as pl
    dims = (96, 128, 256)
    T = synth.gaussian(int(np.prod(dims)), 1, seed=12).reshape(dims)
    Tt = cuda(T)
    for mode in range(3):
        W = to_np(shg.project(Tt, mode, 48, seed=9))
        U = np.ascontiguousarray(pl.unfold(T, mode))
        check_bars(orc, U, orc.omega_f16(U.shape[1], 48, seed=9, stream_id=mode), W)


@pytest.mark.parametrize("m,k,n,mmajor", [(129, 700, 200, False), (1000, 4096, 256, False), (700, 1024, 144, True),
                                          (4096, 512, 128, True)])
def test_cta_pair_mode(shg, orc, m, k, n, mmajor):
    """tcgen05.mma.cta_group::2 mainloop (cluster of 2, Omega halves per CTA) incl. ragged pair tiles."""
    A = synth.gaussian(m, k, seed=m + n)
    Om = shg.gen_omega(k, n, seed=4)
    assert shg.plan(m, n, k, {"pair": 1})["cta_pair"] == 1
    if mmajor:
        Y = to_np(shg.shgemm_at(torch.from_numpy(np.ascontiguousarray(A.T)).cuda(), Om, tune={"pair": 1}))
    else:
        Y = to_np(shg.shgemm(cuda(A), Om, tune={"pair": 1}))
    check_bars(orc, A, omega_bits(Om), Y)



@pytest.mark.parametrize("m,k,n,tune", [(160, 1 << 19, 24, None), (200, 1 << 16, 40, {"a_box": 2}), (300, 4096 + 32, 144, {"a_box": 2, "pair": 1}),
                                        (129, 96, 64, {"a_box": 2}), (300, 4096 + 32, 144, {"a_box": 1, "pair": 1})])
def test_a_box_layouts(shg, orc, m, k, n, tune):
    """Both row-major A staging layouts (two {32 k, 128 rows} boxes, or one {2 x 32 k, 128 rows}
    row-major box, auto-selected for rows >= 2 MiB apart) incl. a k % 64 == 32 tail; a_box 2
    without k % 32 == 0 is rejected."""
    A = synth.gaussian(m, k, seed=k + m)
    om, Y = _run(shg, A, k, n, tune=tune)
    check_bars(orc, A, om, Y)
    with pytest.raises(shg.SHGError):
        shg.shgemm(cuda(synth.gaussian(64, 100, seed=1)), shg.gen_omega(100, 16), tune={"a_box": 2})


def test_omega_multicast_option_removed(shg):
    """Round 2 removed the Omega-multicast instantiations (no steady-state gain):
    omega_mcast 0 / 1 plan normally, 2..4 are rejected instead of silently ignored."""
    assert shg.plan(4096, 256, 512, {"omega_mcast": 1})["omega_mcast"] == 1
    for mc in (2, 3, 4, -1):
        with pytest.raises(shg.SHGError):
            shg.plan(4096, 256, 512, {"omega_mcast": mc})


@pytest.mark.parametrize("m,k,n,tune", [(1000, 1500, 272, None), (600, 777, 288, None), (130, 640, 270, None),
                                        (700, 512, 560, {"bn": 288}), (512, 2048, 272, {"pair": 2}),
                                        (1024, 1024, 300, {"bn": 288})])
@pytest.mark.parametrize("mmajor", [False, True])
def test_wide_tiles(shg, orc, m, k, n, tune, mmajor):
    """256 < BN <= 288 (one N tile for n = 257..288, K_c = 64, 3 chunk slots): the bars, K- and
    M-major A, single CTAs and pairs, ragged n inside the wide tile, two wide tiles."""
    rng = np.random.default_rng(m + k + n)
    A = rng.standard_normal((m, k)).astype(np.float32)
    Om = shg.gen_omega(k, n, seed=2)
    plan = shg.plan(m, n, k, tune)
    assert plan["bn"] in (272, 288) and plan["path"] == 0, plan
    if mmajor:
        Y = shg.shgemm_at(cuda(np.ascontiguousarray(A.T)), Om, tune=tune)
    else:
        Y = shg.shgemm(cuda(A), Om, tune=tune)
    torch.cuda.synchronize()
    check_bars(orc, A, omega_bits(Om), to_np(Y))


def test_wide_tiles_rejected_for_tf32(shg):
    with pytest.raises(shg.SHGError):
        shg.plan(1000, 272, 512, {"bn": 272}, tc="tf32")
    assert shg.plan(1000, 272, 512, tc="tf32")["bn"] <= 256


@pytest.mark.parametrize("k,n,row0,dist", [(1000, 64, 0, 0), (4096, 272, 8, 0), (77, 33, 4, 1), (130, 16, 0, 3)])
def test_omega_tiled_layout_bit_exact(shg, orc, k, n, row0, dist):
    """gen_omega_f16_tiled: element (i, j) at (i//64)*n*64 + j*64 + i%64, same bits as the oracle,
    the last tile's rows beyond k zero."""
    t = to_np(shg.gen_omega_tiled(k, n, seed=11, dist=dist, stream_id=3, row0=row0, k_total=k + row0)).view(np.uint16)
    ref = orc.omega_f16(k, n, seed=11, dist=dist, stream_id=3, row0=row0, k_total=k + row0)   # (k, n)
    kt = (k + 63) // 64
    tiles = t.reshape(kt, n, 64)
    full = np.zeros((kt * 64, n), dtype=np.uint16)
    full[:k] = ref
    np.testing.assert_array_equal(tiles.transpose(0, 2, 1).reshape(kt * 64, n), full)


@pytest.mark.parametrize("m,k,n,tune", [(1024, 4096, 64, None), (700, 1000, 256, None), (300, 640, 272, None),
                                        (128, 8192, 32, None), (512, 1024, 128, {"pair": 2})])
def test_shgemm_tiled_equals_column_major(shg, m, k, n, tune):
    """The k-tiled Omega changes only the TMA box shape: Y bitwise equal to the column-major path."""
    g = torch.Generator(device="cuda").manual_seed(m + n)
    A = torch.randn(m, k, device="cuda", generator=g)
    y_cm = shg.shgemm(A, shg.gen_omega(k, n, seed=5), tune=tune)
    y_t = shg.shgemm_tiled(A, shg.gen_omega_tiled(k, n, seed=5), n, tune=tune)
    torch.cuda.synchronize()
    assert torch.equal(y_cm, y_t)


@pytest.mark.parametrize("G", [2, 3, 8])
def test_row_shards_concatenate_to_unsharded_bitwise(shg, G):
    """§8e verification on one GPU: the G row blocks of the sharded driver (each projected with its
    own regenerated Omega) concatenate to the unsharded Y bit for bit (per-row arithmetic does not
    depend on the tile grid), and every shard's Omega has the same checksum."""
    from paper_2304_04612_b200.shard import checksum_bits, row_partition
    m, k, n = 524288 + 77, 4096, 256
    A = shg.synth("gauss", 2, 0x100, m, k)
    Y = shg.shgemm(A, shg.gen_omega(k, n, seed=0))
    crcs = set()
    for g in range(G):
        r0, rows = row_partition(m, G, g)
        Om = shg.gen_omega(k, n, seed=0)            # regenerated per shard, no communication
        crcs.add(checksum_bits(Om))
        Yg = shg.shgemm(A[r0:r0 + rows], Om)
        torch.cuda.synchronize()
        assert torch.equal(Yg, Y[r0:r0 + rows]), g
    assert len(crcs) == 1


@pytest.mark.parametrize("gen_mode", [1, 2])
@pytest.mark.parametrize("dims,mode,n", [((512, 64, 128), 0, 64), ((512, 64, 128), 1, 48), ((512, 64, 128), 2, 32),
                                         ((300, 40, 100), 0, 64), ((96, 2048, 8), 1, 16)])
def test_project_inkernel_omega_bit_exact(shg, orc, dims, mode, n, gen_mode):
    """project() generates Omega_(mode) inside the mainloop (generator warps, flags per 64-k tile)
    when the plan allows it: the Omega it leaves in the caller's workspace is bit-identical to
    gen_omega_f16_tiled (and the oracle), and W meets the bars. gen_mode 2: the generator warps stay
    idle, so every tile comes from the Omega stagers' generate-on-timeout fallback."""
    from oracle import pipelines as opl
    T = synth.gaussian(int(np.prod(dims)), 1, seed=13).reshape(dims)
    Tc = cuda(T)
    ws = torch.zeros(shg.project_workspace_size(list(dims), mode, n), dtype=torch.uint8, device="cuda")
    prev = shg.get_inkernel_omega()
    shg.set_inkernel_omega(gen_mode)
    try:
        helped = shg.inkernel_omega_fallbacks()
        launches = shg.launch_count()
        W = shg.project(Tc, mode, n, seed=4, workspace=ws)
        torch.cuda.synchronize()
        K = int(np.prod(dims)) // dims[mode]
        expect = 1 + (1 if shg.plan(dims[mode], n, K)["split_k"] > 1 else 0)
        assert shg.launch_count() - launches == expect      # mainloop (+ split-K reduce): no gen_omega launch
        if gen_mode == 2:   # every k-tile came from a stager's fallback (several CTAs may each make one)
            assert shg.inkernel_omega_fallbacks() - helped >= (K + 63) // 64
        else:               # one kernel alone, every CTA resident: the generator warps made every tile
            assert shg.inkernel_omega_fallbacks() == helped
    finally:
        shg.set_inkernel_omega(prev)
    nb = n * ((K + 63) // 64) * 64
    om_ws = to_np(ws[:2 * nb]).view(np.uint16)
    om_ref = to_np(shg.gen_omega_tiled(K, n, seed=4, stream_id=mode)).view(np.uint16)
    np.testing.assert_array_equal(om_ws, om_ref)
    Ai = np.ascontiguousarray(opl.unfold(T, mode))
    check_bars(orc, Ai, orc.omega_f16(K, n, seed=4, stream_id=mode), to_np(W))


def test_project_inkernel_omega_concurrent_streams(shg):
    """Four in-kernel-Omega projections on four streams at once, each of whose plans fills the grid:
    their CTAs cannot all be resident together, so stagers wait on generator CTAs that are not
    scheduled and take the generate-on-timeout fallback. Every W equals the sequential result bit
    for bit (no deadlock, no watchdog trap)."""
    prev = shg.get_inkernel_omega()
    shg.set_inkernel_omega(True)
    try:
        dims, n = (1024, 1024, 512), 64     # 2 GiB each: one call outlasts the 200-us fallback timeout
        Ts = [torch.randn(*dims, device="cuda", generator=torch.Generator(device="cuda").manual_seed(i))
              for i in range(4)]
        ref = [shg.project(T, 0, n, seed=i) for i, T in enumerate(Ts)]
        torch.cuda.synchronize()
        helped = shg.inkernel_omega_fallbacks()
        streams = [torch.cuda.Stream() for _ in Ts]
        outs = [torch.empty_like(r) for r in ref]
        wss = [torch.empty(shg.project_workspace_size(list(dims), 0, n), dtype=torch.uint8, device="cuda")
               for _ in Ts]
        for rep in range(3):
            torch.cuda.synchronize()
            for i, (T, st) in enumerate(zip(Ts, streams)):
                with torch.cuda.stream(st):
                    shg.project(T, 0, n, seed=i, out=outs[i], workspace=wss[i])
            torch.cuda.synchronize()
            for o, r in zip(outs, ref):
                assert torch.equal(o, r)
        print("fallback tiles in the concurrent calls:", shg.inkernel_omega_fallbacks() - helped)
    finally:
        shg.set_inkernel_omega(prev)


def test_project_inkernel_omega_equals_separate_generation(shg, tmp_path):
    """W with in-kernel Omega (SHG_OMGEN=1) == W with the separate generator, bit for bit."""
    import subprocess
    import sys
    code = ("import sys, numpy as np, torch; sys.path.insert(0, %r); import paper_2304_04612_b200 as shg, synth;"
            "T = torch.from_numpy(synth.gaussian(512*64*128, 1, seed=13).reshape(512, 64, 128)).cuda();"
            "np.save(sys.argv[1], np.stack([shg.project(T, md, 64, seed=4).cpu().numpy()[:64] for md in range(3)]))"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    outs = []
    for flag in ("1", "0"):           # SHG_OMGEN sets the process default of shg_set_inkernel_omega
        path = str(tmp_path / f"w{flag}.npy")
        env = dict(os.environ, SHG_OMGEN=flag)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, timeout=300)
        outs.append(np.load(path))
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("dims,mode", [((64, 96, 128), 0), ((64, 96, 128), 1), ((64, 96, 128), 2)])
def test_project_omega_equals_project(shg, dims, mode):
    """project_omega (caller's k-tiled Omega) == project (Omega generated inside), bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(mode)
    T = torch.randn(*dims, device="cuda", generator=g)
    K = T.numel() // dims[mode]
    W1 = shg.project(T, mode, 24, seed=8)
    W2 = shg.project(T, mode, 24, omega=shg.gen_omega_tiled(K, 24, seed=8, stream_id=mode))
    torch.cuda.synchronize()
    assert torch.equal(W1, W2)


@pytest.mark.parametrize("dims,mode", [((24, 40, 96), 1), ((10, 24, 32), 1), ((6, 7, 160, 32), 2), ((50, 8, 96), 0)])
def test_project_slab_views_s_multiple_of_32(shg, orc, dims, mode):
    """Middle-mode unfoldings whose contiguous run S is a multiple of 32 but not of 64 are read in
    place (a 64-k stage's second 32-k half continues in the next slab), no copy: bars vs oracle."""
    from oracle import pipelines as opl
    T = synth.gaussian(int(np.prod(dims)), 1, seed=31).reshape(dims)
    S = int(np.prod(dims[mode + 1:]))
    assert S % 32 == 0
    W = to_np(shg.project(cuda(T), mode, 40, seed=2))
    Ai = np.ascontiguousarray(opl.unfold(T, mode))
    check_bars(orc, Ai, orc.omega_f16(Ai.shape[1], 40, seed=2, stream_id=mode), W)


@pytest.mark.parametrize("m,k,n,tune,mmajor", [(1000, 640, 256, None, False), (1000, 640, 272, None, False),
                                               (100, 640, 64, None, False), (300, 4096, 32, {"split_k": 4}, False),
                                               (1000, 640, 128, None, True), (700, 512, 200, {"pair": 2}, True)])
def test_nonfinite_flag_every_plan(shg, m, k, n, tune, mmajor):
    """The optional non-finite flag across plan shapes (pairs, wide tiles, single CTAs, split-K
    reduce, M-major): one A element >= 65520 in one row poisons exactly that row, flag set; a clean
    A leaves the flag 0."""
    g = torch.Generator(device="cuda").manual_seed(m + n)
    A = torch.randn(m, k, device="cuda", generator=g)
    Om = shg.gen_omega(k, n, seed=1)
    bad = m // 3
    for poison in (False, True):
        if poison:
            A[bad, k // 2] = 70000.0
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        if mmajor:
            Y = shg.shgemm_at(A.t().contiguous(), Om, nonfinite=flag, tune=tune)
        else:
            Y = shg.shgemm(A, Om, nonfinite=flag, tune=tune)
        torch.cuda.synchronize()
        finite_rows = torch.isfinite(Y).all(dim=1)
        if poison:
            assert int(flag.item()) == 1 and not bool(finite_rows[bad])
            finite_rows[bad] = True
            assert bool(finite_rows.all())
        else:
            assert int(flag.item()) == 0 and bool(finite_rows.all())


def test_omega_statistics_1e8(shg):
    """the Gaussian Omega's statistics on >= 1e8 samples (device-generated; bit-identical
    to the oracle's stream, test_omega_bit_exact_1e8): mean 0 and variance 1 within 5 sigma_MC of the
    FP16-rounded N(0,1) truncated at |z| <= 5.77 (OMEGA_SPEC), kurtosis 3, symmetry of the signs, and
    the FP16-subnormal-or-zero rate 2 phi(0) 2^-14 = 4.87e-5 (reading c4-20)."""
    import math
    n_tot, s1, s2, s4, neg, sub = 0, 0.0, 0.0, 0.0, 0, 0
    for stream in range(2):
        Om = shg.gen_omega(1 << 20, 64, seed=99, stream_id=stream, layout="row")    # 2^26 per stream
        z = Om.double().flatten()
        n_tot += z.numel()
        s1 += float(z.sum())
        s2 += float((z * z).sum())
        s4 += float((z ** 4).sum())
        neg += int((z < 0).sum())
        sub += int(((Om.view(torch.int16) & 0x7C00) == 0).sum())
    assert n_tot >= 1e8
    mean, var = s1 / n_tot, s2 / n_tot
    kurt = (s4 / n_tot) / var ** 2
    assert abs(mean) < 5.0 / math.sqrt(n_tot), mean
    assert abs(var - 1.0) < 5.0 * math.sqrt(2.0 / n_tot) + 1e-6, var      # + FP16 rounding of the draws
    assert abs(kurt - 3.0) < 5.0 * math.sqrt(24.0 / n_tot) + 1e-4, kurt
    assert abs(neg / n_tot - 0.5) < 5.0 * 0.5 / math.sqrt(n_tot), neg / n_tot
    p = 2.0 / math.sqrt(2 * math.pi) * 2.0 ** -14
    assert abs(sub / n_tot - p) < 5.0 * math.sqrt(p / n_tot), sub / n_tot


@pytest.mark.parametrize("dist", ["normal", "uniform"])
@pytest.mark.parametrize("k", [16, 64, 256, 1024, 4096])
def test_elementwise_bar_100_trials(shg, orc, dist, k):
    """SURVEY c6 "Bounds": the elementwise bar of c5 (P:594-597 plus the split term) and the
    Frobenius bars hold in 100 trials per k for both A distributions of the paper's accuracy
    experiment (A ~ N(0,1) and U(0,1); Gaussian Omega), 64 x k x 32 each."""
    m, n = 64, 32
    worst = 0.0
    for t in range(100):
        A = synth.gaussian(m, k, seed=7000 + t) if dist == "normal" else synth.uniform(m, k, seed=7000 + t)
        om, Y = _run(shg, A, k, n, seed=t)
        _, _, w = check_bars(orc, A, om, Y)
        worst = max(worst, w)
    assert worst <= 1.0
