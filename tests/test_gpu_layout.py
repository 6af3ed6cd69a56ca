"""Omega layouts at the boundary (include/shgemm.h): row-major Omega (ldo >= n, the
layout of shgemm()/gen_omega_f16()) and column-major Omega (ldo >= k, the tensor cores' K-major
operand) give BITWISE-identical Y on every path (FP16 and TF32 tensor cores, CTA pairs, split-K,
wide tiles, M-major A, the CUDA-core fallback, host streaming); gen_omega_f16 writes the same bits
in both layouts (and the oracle's). Also shgemm_host with a short last chunk and from concurrent
host threads."""
import ctypes
import threading

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


@pytest.mark.parametrize("k,n,seed,dist,row0", [(512, 32, 0, 0, 0), (1001, 17, 5, 0, 3), (4096, 256, 0, 0, 0),
                                                 (333, 70, 2, 1, 0), (2000, 40, 9, 3, 8)])
def test_gen_omega_row_major_bits(shg, orc, k, n, seed, dist, row0):
    row = shg.gen_omega(k, n, seed=seed, dist=dist, row0=row0, layout="row")
    col = shg.gen_omega(k, n, seed=seed, dist=dist, row0=row0)
    assert row.stride() == (n, 1) and col.stride(0) == 1
    ref = orc.omega_f16(k, n, seed=seed, dist=dist, row0=row0, k_total=k)
    assert np.array_equal(omega_bits(row), ref)
    assert np.array_equal(omega_bits(col), ref)


def test_gen_omega_f16_c_abi_row_major_padded_ldo(shg, orc):
    """gen_omega_f16 (§8(b) signature): row-major with ldo > n; padding columns untouched."""
    k, n, ldo = 777, 50, 64
    buf = torch.full((k, ldo), -1, dtype=torch.int16, device="cuda")
    L = shg.lib()
    assert L.gen_omega_f16(k, n, 11, 0, ctypes.c_void_p(buf.data_ptr()), ldo, shg._stream()) == 0
    torch.cuda.synchronize()
    got = to_np(buf).view(np.uint16)
    assert np.array_equal(got[:, :n], orc.omega_f16(k, n, seed=11))
    assert np.all(got[:, n:] == 0xFFFF)


def _row_copy(Om, pad=0):
    k, n = Om.shape
    buf = torch.zeros((k, n + pad), dtype=torch.float16, device="cuda")
    buf[:, :n] = Om
    return buf[:, :n]


@pytest.mark.parametrize("m,k,n,tune", [
    (512, 512, 32, None),                           # config 1 shape
    (1000, 777, 48, None),                          # ragged
    (700, 3000, 256, None),                         # CTA pairs
    (300, 5000, 64, {"split_k": 3}),                # split-K
    (600, 1024, 272, None),                         # wide tile
    (513, 640, 100, {"pair": 2}),
    (400, 1000, 96, {"tc": "tf32"}),                # SHGEMM-TF32 (widening reads either layout)
    (257, 300, 40, {"force_simt": 1}),              # CUDA-core fallback
])
def test_shgemm_row_major_equals_column_major_bitwise(shg, orc, m, k, n, tune):
    g = torch.Generator(device="cuda").manual_seed(m + k + n)
    A = torch.randn(m, k, device="cuda", generator=g)
    col = shg.gen_omega(k, n, seed=3)
    row = _row_copy(col, pad=5)                     # ldo = n + 5 (not a multiple of 8: copied anyway)
    assert shg.omega_layout(row) == (shg.OMEGA_ROW_MAJOR, n + 5)
    y_col = shg.shgemm(A, col, tune=tune)
    y_row = shg.shgemm(A, row, tune=tune)
    torch.cuda.synchronize()
    assert torch.equal(y_col, y_row)
    if m * k <= 2e6:
        check_bars(orc, to_np(A), omega_bits(col), to_np(y_row))


def test_shgemm_c_abi_row_major(shg, orc):
    """The §8(b) call itself: shgemm(m, n, k, A, lda, Omega, ldo >= n, Y, ldc, stream) on a row-major
    Omega from gen_omega_f16, against the oracle, and equal to the column-major _ex call."""
    m, k, n = 1000, 777, 48
    L = shg.lib()
    A = shg.synth("gauss", 9, 0x100, m, k)
    Om = torch.empty((k, n), dtype=torch.float16, device="cuda")
    p = lambda t: ctypes.c_void_p(t.data_ptr())
    assert L.gen_omega_f16(k, n, 0, 0, p(Om), n, shg._stream()) == 0
    Y = torch.empty((m, n), device="cuda")
    assert L.shgemm(m, n, k, p(A), k, p(Om), n, p(Y), n, shg._stream()) == 0
    torch.cuda.synchronize()
    check_bars(orc, to_np(A), omega_bits(Om), to_np(Y))
    assert torch.equal(Y, shg.shgemm(A, shg.gen_omega(k, n, seed=0)))


def test_shgemm_at_row_major(shg):
    g = torch.Generator(device="cuda").manual_seed(3)
    At = torch.randn(900, 640, device="cuda", generator=g)     # A = At^T: m = 640, k = 900
    col = shg.gen_omega(900, 64, seed=1)
    assert torch.equal(shg.shgemm_at(At, col), shg.shgemm_at(At, _row_copy(col)))


@pytest.mark.parametrize("layout", ["row", "col"])
def test_shgemm_host_short_last_chunk(shg, layout):
    """shgemm_host with m not a multiple of the chunk: the workspace covers the short last chunk's
    plan (8960 x 8192 x 256 with chunk 8192 rows needs more split-K scratch for the
    768-row tail than for a full chunk); Y equals the device-resident shgemm bitwise."""
    m, k, n, chunk = 8960, 8192, 256, 8192
    A = shg.synth("gauss", 4, 0x100, m, k)
    Om = shg.gen_omega(k, n, seed=2, layout=layout)
    ws = torch.empty(shg.host_workspace_size(n, k, chunk, layout=layout), dtype=torch.uint8, device="cuda")
    Y_h = shg.shgemm_host(A.cpu().pin_memory(), Om, chunk_rows=chunk, workspace=ws)
    torch.cuda.synchronize()
    ref = torch.cat([shg.shgemm(A[:chunk], Om), shg.shgemm(A[chunk:], Om)])
    assert torch.equal(Y_h, ref.cpu())


def test_shgemm_host_threads(shg):
    """Four host threads call shgemm_host concurrently on their own streams (per-call side streams
    and events): every result equals the serial one bitwise."""
    m, k, n = 3000, 1024, 64
    A = shg.synth("gauss", 5, 0x100, m, k).cpu().pin_memory()
    Om = shg.gen_omega(k, n, seed=7)
    ref = shg.shgemm_host(A, Om, chunk_rows=1024)
    torch.cuda.synchronize()
    outs, err = [None] * 4, []

    def worker(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    outs[t] = shg.shgemm_host(A, Om if t % 2 else _row_copy(Om), chunk_rows=1024, stream=s)
            s.synchronize()
        except Exception as e:   # surfaced below
            err.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not err, err
    for t in range(4):
        assert torch.equal(outs[t], ref), t


@pytest.mark.parametrize("k,n", [(1, 64), (1, 1), (40, 1), (1, 300), (7, 1)])
@pytest.mark.parametrize("layout", ["row", "col"])
def test_degenerate_omega_shapes(shg, orc, k, n, layout):
    """k = 1 or n = 1 in both layouts: the binding passes the real stride as ldo (a (1, n)
    column-major view has strides (1, ldo)); found by the round-2 fuzz."""
    g = torch.Generator(device="cuda").manual_seed(k * 1000 + n)
    A = torch.randn(300, k, device="cuda", generator=g)
    Om = shg.gen_omega(k, n, seed=3, layout=layout)
    Y = shg.shgemm(A, Om)
    Yt = shg.shgemm_at(A.t().contiguous(), Om)
    torch.cuda.synchronize()
    ref = to_np(A).astype(np.float64) @ orc.f16_bits_as_float(omega_bits(Om)).astype(np.float64)
    np.testing.assert_allclose(to_np(Y), ref, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(to_np(Yt), ref, rtol=1e-6, atol=1e-6)
