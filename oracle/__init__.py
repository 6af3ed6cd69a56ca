"""CPU oracle for the SHGEMM random projection (arxiv 2304.04612).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The product path
(``paper_2304_04612_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, fp64/fp32, built with
``-ffp-contract=off``); this module only loads it and marshals numpy arrays. The RandNLA
pipelines (Alg 1 and Alg 2 of the paper) are in ``oracle/pipelines.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

GAUSSIAN, RADEMACHER, SPARSE3, VERYSPARSE = 0, 1, 2, 3
DIST_IDS = {"gaussian": 0, "rademacher": 1, "sparse3": 2, "verysparse": 3}


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2 -ffp-contract=off, OpenMP)."""
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC):
        return _LIB_PATH
    cmd = ["gcc", "-O2", "-mfma", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
           "-shared", "-std=c11", "-Wall", "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            i64, u64, u32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
            L.orc_philox4x32_10.argtypes = [vp, vp, vp]
            L.orc_f32_to_f16_rn.argtypes = [ctypes.c_float]
            L.orc_f32_to_f16_rn.restype = ctypes.c_uint16
            L.orc_f16_to_f32.argtypes = [ctypes.c_uint16]
            L.orc_f16_to_f32.restype = ctypes.c_float
            L.orc_ln_spec.argtypes = [u32]
            L.orc_ln_spec.restype = ctypes.c_float
            L.orc_radius_spec.argtypes = [u32]
            L.orc_radius_spec.restype = ctypes.c_float
            L.orc_sincos_spec.argtypes = [u32, vp, vp]
            L.orc_sparse_threshold.argtypes = [ctypes.c_int, i64]
            L.orc_sparse_threshold.restype = u32
            L.orc_omega_element.argtypes = [u64, u32, ctypes.c_int, i64, u64, u32]
            L.orc_omega_element.restype = ctypes.c_uint16
            L.orc_omega_f16.argtypes = [i64, i64, u64, u32, i64, ctypes.c_int, i64, vp, i64]
            L.orc_split.argtypes = [vp, i64, vp, vp]
            L.orc_split_tf32.argtypes = [vp, i64, vp, vp]
            L.orc_f32_to_tf32_rn.argtypes = [ctypes.c_float]
            L.orc_f32_to_tf32_rn.restype = u32
            for name in ("orc_gemm_y64", "orc_gemm_y32", "orc_gemm_ysplit64", "orc_gemm_ysplit64_tf32",
                         "orc_gemm_y64_f32b", "orc_gemm_y32_f32b", "orc_gemm_ytcec64"):
                getattr(L, name).argtypes = [i64, vp, i64, i64, vp, i64, vp, i64, vp, i64]
            L.orc_gauss_f32.argtypes = [u64, u32, u64, u64]
            L.orc_gauss_f32.restype = ctypes.c_float
            L.orc_unif_f32.argtypes = [u64, u32, u64, u64]
            L.orc_unif_f32.restype = ctypes.c_float
            L.orc_synth_rows_f32.argtypes = [ctypes.c_int, u64, u32, i64, vp, i64, vp]
            L.orc_num_threads.restype = ctypes.c_int
            L.orc_ln_spec_batch.argtypes = [vp, i64, vp]
            L.orc_sincos_spec_batch.argtypes = [vp, i64, vp, vp]
            L.orc_radius_spec_batch.argtypes = [vp, i64, vp]
            L.orc_f32_to_f16_batch.argtypes = [vp, i64, vp]
            L.orc_gauss_column_f32.argtypes = [u64, u32, u32, i64, i64, vp]
            _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().orc_num_threads())


# --------------------------------------------------------------------------- Philox / Box–Muller
def philox4x32_10(ctr, key) -> tuple:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return tuple(int(v) for v in out)


def ln_spec(na: int) -> float:
    return float(lib().orc_ln_spec(int(na)))


def radius_spec(xa: int) -> float:
    return float(lib().orc_radius_spec(int(xa)))


def sincos_spec(xb: int):
    c = ctypes.c_float()
    s = ctypes.c_float()
    lib().orc_sincos_spec(int(xb), ctypes.byref(c), ctypes.byref(s))
    return float(c.value), float(s.value)


# --------------------------------------------------------------------------- FP16 / split
def ln_spec_batch(na: np.ndarray) -> np.ndarray:
    na = np.ascontiguousarray(na, dtype=np.uint32)
    out = np.empty(na.size, dtype=np.float32)
    lib().orc_ln_spec_batch(_ptr(na), na.size, _ptr(out))
    return out


def radius_spec_batch(xa: np.ndarray) -> np.ndarray:
    xa = np.ascontiguousarray(xa, dtype=np.uint32)
    out = np.empty(xa.size, dtype=np.float32)
    lib().orc_radius_spec_batch(_ptr(xa), xa.size, _ptr(out))
    return out


def sincos_spec_batch(xb: np.ndarray):
    xb = np.ascontiguousarray(xb, dtype=np.uint32)
    c = np.empty(xb.size, dtype=np.float32)
    s = np.empty(xb.size, dtype=np.float32)
    lib().orc_sincos_spec_batch(_ptr(xb), xb.size, _ptr(c), _ptr(s))
    return c, s


def gauss_column_f32(seed: int, stream_id: int, j: int, row0: int, count: int) -> np.ndarray:
    """Pre-rounding binary32 Gaussian values z of column j (OMEGA_SPEC §3)."""
    out = np.empty(count, dtype=np.float32)
    lib().orc_gauss_column_f32(seed, stream_id, j, row0, count, _ptr(out))
    return out


def f32_to_f16_batch(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint16)
    lib().orc_f32_to_f16_batch(_ptr(x), x.size, _ptr(out))
    return out


def f32_to_f16_bits(x: float) -> int:
    return int(lib().orc_f32_to_f16_rn(float(np.float32(x))))


def f16_bits_to_f32(h: int) -> float:
    return float(lib().orc_f16_to_f32(int(h)))


def split(a: np.ndarray):
    """Eqs 14-15. Returns (hi_bits, lo_bits) as uint16 arrays."""
    a = np.ascontiguousarray(a, dtype=np.float32).reshape(-1)
    hi = np.empty(a.size, dtype=np.uint16)
    lo = np.empty(a.size, dtype=np.uint16)
    lib().orc_split(_ptr(a), a.size, _ptr(hi), _ptr(lo))
    return hi, lo


def split_tf32(a: np.ndarray):
    """Eqs 14-15 with toLow = TF32 (SHGEMM-TF32). Returns (hi_bits, lo_bits) as uint32
    FP32 bit patterns (low 13 bits zero)."""
    a = np.ascontiguousarray(a, dtype=np.float32).reshape(-1)
    hi = np.empty(a.size, dtype=np.uint32)
    lo = np.empty(a.size, dtype=np.uint32)
    lib().orc_split_tf32(_ptr(a), a.size, _ptr(hi), _ptr(lo))
    return hi, lo


def f32_to_tf32_bits(x: float) -> int:
    return int(lib().orc_f32_to_tf32_rn(float(x)))


# --------------------------------------------------------------------------- Ω
def sparse_threshold(dist: int, k_total: int) -> int:
    return int(lib().orc_sparse_threshold(int(dist), int(k_total)))


def omega_element(seed: int, stream_id: int, dist: int, k_total: int, i: int, j: int) -> int:
    return int(lib().orc_omega_element(seed, stream_id, dist, k_total, i, j))


def omega_f16(k: int, n: int, seed: int = 0, dist: int = GAUSSIAN, stream_id: int = 0,
              row0: int = 0, k_total: int | None = None) -> np.ndarray:
    """Ω as FP16 bits, returned as a (k, n) uint16 array (logical layout; OMEGA_SPEC §5)."""
    if isinstance(dist, str):
        dist = DIST_IDS[dist]
    k_total = k if k_total is None else k_total
    buf = np.empty((n, k), dtype=np.uint16)  # column-major k x n == row-major n x k
    if k and n:
        lib().orc_omega_f16(k, n, seed, stream_id, row0, dist, k_total, _ptr(buf), k)
    return buf.T


def f16_bits_as_float(bits: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(bits, dtype=np.uint16).view(np.float16).astype(np.float32)


# --------------------------------------------------------------------------- GEMMs
def _gemm(fn, out_dtype, A, omega_bits, rows=None):
    A = np.ascontiguousarray(A, dtype=np.float32)
    m, k = A.shape
    k2, n = omega_bits.shape
    assert k2 == k
    om = np.ascontiguousarray(np.asarray(omega_bits, dtype=np.uint16).T)  # n x k == column-major
    if rows is None:
        nrows, rp = m, None
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        nrows, rp = rows.size, _ptr(rows)
    Y = np.zeros((nrows, n), dtype=out_dtype)
    if nrows and n:
        fn(nrows, rp, n, k, _ptr(A), k, _ptr(om), k, _ptr(Y), n)
    return Y


def gemm_y64(A, omega_bits, rows=None) -> np.ndarray:
    """C_F64 of Fig 5: exact products, fp64 sum ascending in l."""
    return _gemm(lib().orc_gemm_y64, np.float64, A, omega_bits, rows)


def gemm_y32(A, omega_bits, rows=None) -> np.ndarray:
    """Naive FP32: acc = fmaf(a, w, acc) sequentially in l (SGEMM comparator)."""
    return _gemm(lib().orc_gemm_y32, np.float32, A, omega_bits, rows)


def gemm_ysplit64(A, omega_bits, rows=None) -> np.ndarray:
    """Eq 16 in FP64: sum_l (hi + lo 2^-11) w."""
    return _gemm(lib().orc_gemm_ysplit64, np.float64, A, omega_bits, rows)


def gemm_ysplit64_tf32(A, omega_bits, rows=None) -> np.ndarray:
    """Eq 16 in FP64 with the TF32 split of SHGEMM-TF32."""
    return _gemm(lib().orc_gemm_ysplit64_tf32, np.float64, A, omega_bits, rows)


def _gemm_f32b(fn, out_dtype, A, B, rows=None):
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.asarray(B, dtype=np.float32)
    m, k = A.shape
    k2, n = B.shape
    assert k2 == k
    bc = np.ascontiguousarray(B.T)          # n x k == column-major k x n
    if rows is None:
        nrows, rp = m, None
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        nrows, rp = rows.size, _ptr(rows)
    Y = np.zeros((nrows, n), dtype=out_dtype)
    if nrows and n:
        fn(nrows, rp, n, k, _ptr(A), k, _ptr(bc), k, _ptr(Y), n)
    return Y


def gemm_y64_f32b(A, B, rows=None) -> np.ndarray:
    """sum_l (double)A[i][l] * (double)B[l][j] for FP32 A and B (exact products), l ascending."""
    return _gemm_f32b(lib().orc_gemm_y64_f32b, np.float64, A, B, rows)


def gemm_y32_f32b(A, B, rows=None) -> np.ndarray:
    """Naive FP32 SGEMM: acc = fmaf(a, b, acc), l ascending (the SGEMM baseline of P:613)."""
    return _gemm_f32b(lib().orc_gemm_y32_f32b, np.float32, A, B, rows)


def gemm_ytcec64(A, B, rows=None) -> np.ndarray:
    """TCEC-SGEMM, Eq 9 in FP64: A_low B_low + (dA_low B_low + A_low dB_low) 2^-11."""
    return _gemm_f32b(lib().orc_gemm_ytcec64, np.float64, A, B, rows)


def relative_error(C, C_ref) -> float:
    """||C - C_ref||_F / ||C_ref||_F in fp64."""
    C = np.asarray(C, dtype=np.float64)
    C_ref = np.asarray(C_ref, dtype=np.float64)
    return float(np.linalg.norm(C - C_ref) / np.linalg.norm(C_ref))


# --------------------------------------------------------------------------- synthetic rows
def synth_rows(kind: str, seed: int, stream_id: int, rows, k: int) -> np.ndarray:
    """Rows of the counter-based synthetic matrix (OMEGA_SPEC §6); kind 'gauss' | 'unif'."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty((rows.size, k), dtype=np.float32)
    if rows.size and k:
        lib().orc_synth_rows_f32(0 if kind == "gauss" else 1, seed, stream_id, rows.size,
                                 _ptr(rows), k, _ptr(out))
    return out
