"""SHGEMM random projection for B200 (sm_100a) — Python binding of libshgemm.so.

Paper: Ootomo & Yokota, "Mixed-precision random projection for RandNLA on Tensor Cores"
(arXiv 2304.04612). The library computes Y = A . Omega (Eq 1) with A in FP32
and Omega in FP16 by SHGEMM (Eqs 14-17) in hand-written tcgen05 CUDA.

This module only marshals arguments (torch tensors -> device pointers, the current CUDA stream)
into the C ABI of include/shgemm.h. Every step of the path runs in the library's kernels; there
is no CPU or PyTorch fallback — if libshgemm.so is missing or the device is not a B200 the calls
raise.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

__all__ = ["shgemm", "shgemm_at", "shgemm_tiled", "shgemm_host", "tcec_sgemm", "tcec_plan", "tcec_workspace_size",
           "gen_omega", "gen_omega_tiled", "project", "project_workspace_size", "set_inkernel_omega", "get_inkernel_omega", "split",
           "split_tf32", "synth", "plan", "workspace_size", "launch_count", "device_supported", "version", "lib",
           "probe_umma", "SHGError", "DISTS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libshgemm.so")
DISTS = {"gaussian": 0, "rademacher": 1, "sparse3": 2, "verysparse": 3}
_STATUS = {0: "SHG_OK", 1: "SHG_ERR_INVALID_VALUE", 2: "SHG_ERR_UNSUPPORTED_DEVICE", 3: "SHG_ERR_CUDA",
           4: "SHG_ERR_WORKSPACE"}
_lock = threading.Lock()
_lib = None


class SHGError(RuntimeError):
    pass


class Tune(ctypes.Structure):
    _fields_ = [("bn", ctypes.c_int32), ("split_k", ctypes.c_int32), ("max_ctas", ctypes.c_int32),
                ("force_simt", ctypes.c_int32), ("debug_flags", ctypes.c_int32), ("pair", ctypes.c_int32),
                ("a_box", ctypes.c_int32), ("tc", ctypes.c_int32), ("omega_mcast", ctypes.c_int32),
                ("prof", ctypes.c_void_p), ("omega_layout", ctypes.c_int32), ("stream_k", ctypes.c_int32),
                ("a_mcast", ctypes.c_int32)]


class Plan(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("bn", ctypes.c_int32), ("n_tiles", ctypes.c_int32),
                ("m_tiles", ctypes.c_int32), ("split_k", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("stages_a", ctypes.c_int32), ("stages_b", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("kernels", ctypes.c_int32), ("cta_pair", ctypes.c_int32), ("tc", ctypes.c_int32),
                ("omega_mcast", ctypes.c_int32), ("stream_k", ctypes.c_int32), ("workspace_bytes", ctypes.c_int64),
                ("a_mcast", ctypes.c_int32)]


def lib():
    """Load libshgemm.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise SHGError(f"{LIB_PATH} is not built (run `python __graft_entry__.py` / build())")
            L = ctypes.CDLL(LIB_PATH)
            i32, i64, u32, u64, vp, sz = (ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                          ctypes.c_void_p, ctypes.c_size_t)
            L.shgemm.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, vp]
            L.shgemm_ex.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ctypes.POINTER(Tune), vp, sz, vp, vp]
            L.shg_workspace_size.argtypes = [i64, i64, i64, ctypes.POINTER(Tune)]
            L.shg_workspace_size.restype = sz
            L.shg_plan.argtypes = [i64, i64, i64, ctypes.POINTER(Tune), ctypes.POINTER(Plan)]
            L.gen_omega_f16.argtypes = [i64, i64, u64, i32, vp, i64, vp]
            L.gen_omega_f16_ex.argtypes = [i64, i64, u64, i32, u32, i64, i64, vp, i64, i32, vp]
            L.project.argtypes = [vp, i32, vp, i32, i64, u64, i32, vp, i64, vp, sz, vp]
            L.shg_project_workspace_size.argtypes = [i32, vp, i32, i64]
            L.shg_project_workspace_size.restype = sz
            L.shgemm_at.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ctypes.POINTER(Tune), vp, sz, vp, vp]
            L.shgemm_host.argtypes = [i64, i64, i64, vp, i64, vp, i64, i32, vp, i64, i64, vp, sz, vp]
            L.shg_host_workspace_size.argtypes = [i64, i64, i64, i32]
            L.shg_host_workspace_size.restype = sz
            L.shg_debug_split.argtypes = [vp, i64, vp, vp, vp]
            L.shg_synth_f32.argtypes = [i32, u64, u32, i64, i64, i64, vp, i64, vp]
            L.shgemm_tf32.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, vp]
            L.project_ex.argtypes = [vp, i32, vp, i32, i64, u64, i32, i32, vp, i64, vp, sz, vp]
            L.shg_project_workspace_size_ex.argtypes = [i32, vp, i32, i64, i32]
            L.project_shard.argtypes = [vp, i32, vp, i32, i64, u64, i32, i32, i64, i64, vp, i64, vp, sz, vp]
            L.gen_omega_f16_tiled.argtypes = [i64, i64, u64, i32, u32, i64, i64, vp, vp]
            L.project_omega.argtypes = [vp, i32, vp, i32, i64, vp, vp, i64, vp, sz, vp]
            L.shgemm_tiled.argtypes = [i64, i64, i64, vp, i64, vp, vp, i64, ctypes.POINTER(Tune), vp, sz, vp, vp]
            L.shg_project_workspace_size_ex.restype = sz
            L.shg_debug_split_tf32.argtypes = [vp, i64, vp, vp, vp]
            L.shg_probe_tma_read.argtypes = [vp, i64, i64, i64, i32, i32, i32, i32, i32, vp, vp]
            L.tcec_sgemm.argtypes = [i64, i64, i64, vp, i64, i32, vp, i64, i32, vp, i64, vp]
            L.tcec_sgemm_ex.argtypes = [i64, i64, i64, vp, i64, i32, vp, i64, i32, vp, i64, ctypes.POINTER(Tune), vp,
                                        sz, vp]
            L.tcec_sgemm_workspace_size.argtypes = [i64, i64, i64, ctypes.POINTER(Tune)]
            L.tcec_sgemm_workspace_size.restype = sz
            L.tcec_plan.argtypes = [i64, i64, i64, ctypes.POINTER(Tune), ctypes.POINTER(Plan)]
            L.shg_launch_count.restype = u64
            L.shg_probe_boxmuller.argtypes = [vp, i64, vp, vp, vp, vp]
            L.shg_set_inkernel_omega.argtypes = [i32]
            L.shg_set_inkernel_omega.restype = None
            L.shg_get_inkernel_omega.argtypes = []
            L.shg_get_inkernel_omega.restype = i32
            L.shg_inkernel_omega_fallbacks.argtypes = []
            L.shg_inkernel_omega_fallbacks.restype = ctypes.c_uint64
            L.shg_set_a_mcast.argtypes = [i32]
            L.shg_set_a_mcast.restype = i32
            L.shg_last_error.restype = ctypes.c_char_p
            L.shg_device_supported.restype = i32
            L.shg_version.restype = ctypes.c_char_p
            L.shg_probe_umma.argtypes = [vp, vp, i32, vp, i32, i32, vp, vp]
            L.shg_probe_mma_rate.argtypes = [i32, i32, i32, i32, vp, i32, vp]
            L.shg_probe_mma_rate.restype = i32
            L.shg_probe_mma2_rate.argtypes = [i32, i32, i32, vp, i32, vp]
            L.shg_probe_mma2_rate.restype = i32
            for name in ("shgemm", "shgemm_ex", "shgemm_at", "shgemm_host", "shg_plan", "gen_omega_f16", "gen_omega_f16_ex", "project",
                         "shg_debug_split", "shg_synth_f32", "shg_probe_umma", "shgemm_tf32", "project_ex",
                         "shg_debug_split_tf32", "tcec_sgemm", "tcec_sgemm_ex", "tcec_plan", "project_shard",
                         "gen_omega_f16_tiled", "shgemm_tiled", "project_omega"):
                getattr(L, name).restype = i32
            _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        msg = lib().shg_last_error().decode()
        raise SHGError(f"{what}: {_STATUS.get(status, status)} {msg}")


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _p(t: torch.Tensor | None):
    """Device pointer of a tensor on the current CUDA device (the library launches there)."""
    if t is None:
        return ctypes.c_void_p(0)
    if not t.is_cuda:
        raise ValueError(f"expected a CUDA tensor, got one on {t.device}")
    if t.device.index != torch.cuda.current_device():
        raise ValueError(f"tensor on {t.device} but the current device is cuda:{torch.cuda.current_device()}")
    return ctypes.c_void_p(t.data_ptr())


def _h(t: torch.Tensor | None):
    """Host pointer (shgemm_host's A and Y)."""
    if t is not None and t.device.type != "cpu":
        raise ValueError(f"expected a host tensor, got one on {t.device}")
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _dist(d) -> int:
    return DISTS[d] if isinstance(d, str) else int(d)


def set_inkernel_omega(on) -> None:
    """project(): generate Omega inside the projection kernel (C ABI shg_set_inkernel_omega; on by
    default). on = 2 is the tests' mode in which every tile comes from the stagers' fallback."""
    lib().shg_set_inkernel_omega(2 if on == 2 else (1 if on else 0))


def get_inkernel_omega() -> int:
    """The current in-kernel Omega setting (0 off, 1 on, 2 fallback-only test mode)."""
    return int(lib().shg_get_inkernel_omega())


def inkernel_omega_fallbacks() -> int:
    """Omega k-tiles generated so far by the stagers' generate-on-timeout fallback (test support)."""
    return int(lib().shg_inkernel_omega_fallbacks())


def set_a_mcast(npa: int) -> int:
    """Process-wide default A multicast (C ABI shg_set_a_mcast): 0 auto, 1 off, 2 / 4 pairs per
    cluster where eligible. Returns the previous value."""
    prev = lib().shg_set_a_mcast(int(npa))
    if prev < 0:
        raise ValueError("npa must be 0, 1, 2 or 4")
    return prev


def launch_count() -> int:
    """Kernels this process has launched through the library (monotonic)."""
    return int(lib().shg_launch_count())


def device_supported() -> bool:
    return bool(lib().shg_device_supported())


def version() -> str:
    return lib().shg_version().decode()


# ----------------------------------------------------------------------------------------- Omega
# shg_omega_layout_t (include/shgemm.h): Omega k x n row-major (ldo >= n) or column-major
# (ldo >= k, the tensor cores' K-major operand, no transpose pass)
OMEGA_ROW_MAJOR, OMEGA_COL_MAJOR = 0, 1
_LAYOUTS = {"row": OMEGA_ROW_MAJOR, "col": OMEGA_COL_MAJOR}


def omega_layout(Omega: torch.Tensor):
    """(shg_omega_layout_t, ldo) of a (k, n) float16 tensor for the C ABI: column-major if
    stride(0) == 1, row-major if stride(1) == 1; the layout is passed explicitly, never inferred
    from ldo by the library."""
    k, n = Omega.shape
    s0, s1 = Omega.stride()
    if k <= 1 and n <= 1:
        return OMEGA_COL_MAJOR, max(k, 1)
    if k <= 1:     # one row: element (0, j) at j * s1 -> row-major if s1 == 1, else column-major, ldo = s1
        return (OMEGA_ROW_MAJOR, max(n, 1)) if s1 == 1 else (OMEGA_COL_MAJOR, s1)
    if n <= 1:     # one column: element (i, 0) at i * s0 -> column-major if s0 == 1, else row-major, ldo = s0
        return (OMEGA_COL_MAJOR, max(k, 1)) if s0 == 1 else (OMEGA_ROW_MAJOR, s0)
    if s0 == 1:
        return OMEGA_COL_MAJOR, s1
    if s1 == 1:
        return OMEGA_ROW_MAJOR, s0
    raise ValueError(f"Omega must have one contiguous dimension (strides {Omega.stride()})")


def gen_omega(k: int, n: int, seed: int = 0, dist="gaussian", stream_id: int = 0, row0: int = 0,
              k_total: int | None = None, device=None, stream=None, out: torch.Tensor | None = None,
              layout: str = "col") -> torch.Tensor:
    """Omega (k x n, FP16) of OMEGA_SPEC.md. layout='col' (default): a column-major view (strides
    (1, ldo), ldo = k rounded up to 8: the layout the tensor cores stream without a copy);
    layout='row': a row-major (k, n) tensor (SURVEY §8(b)'s). With `out` (a (k, n) float16 tensor,
    either layout) the values are written there."""
    if out is None:
        device = torch.device("cuda") if device is None else torch.device(device)
        if layout == "row":
            out = torch.empty((k, n), dtype=torch.float16, device=device)
        elif layout == "col":
            ldo = (k + 7) // 8 * 8 if k > 0 else 8
            out = torch.empty((n, ldo), dtype=torch.float16, device=device)[:, :k].t()
        else:
            raise ValueError("layout must be 'row' or 'col'")
    elif out.dtype != torch.float16 or tuple(out.shape) != (k, n):
        raise ValueError("out must be a (k, n) float16 tensor")
    lay, ldo = omega_layout(out)
    _check(lib().gen_omega_f16_ex(k, n, seed & (2 ** 64 - 1), _dist(dist), stream_id, row0,
                                  k if k_total is None else k_total, _p(out), ldo, lay, _stream(stream)),
           "gen_omega_f16_ex")
    return out


def gen_omega_tiled(k: int, n: int, seed: int = 0, dist="gaussian", stream_id: int = 0, row0: int = 0,
                    k_total: int | None = None, device=None, stream=None) -> torch.Tensor:
    """Omega in the k-tiled layout project() streams (include/shgemm.h gen_omega_f16_tiled): a flat
    float16 tensor of ceil(k/64) * n * 64 elements, element (i, j) at (i//64)*n*64 + j*64 + i%64."""
    device = torch.device("cuda") if device is None else torch.device(device)
    buf = torch.empty(((k + 63) // 64) * n * 64, dtype=torch.float16, device=device)
    _check(lib().gen_omega_f16_tiled(k, n, seed & (2 ** 64 - 1), _dist(dist), stream_id, row0,
                                     k if k_total is None else k_total, _p(buf), _stream(stream)),
           "gen_omega_f16_tiled")
    return buf


def _ld(t: torch.Tensor, rows: int, cols: int) -> int:
    """Leading dimension of a row-major (rows, cols) tensor for the C ABI: its row stride, also for a
    single row when that stride is a valid pitch (a 1-row slice of a padded matrix keeps its 16-B
    aligned pitch and with it the tensor-core path), else max(cols, 1)."""
    s0 = t.stride(0)
    return s0 if (rows > 1 or s0 >= max(cols, 1)) else max(cols, 1)


def _check_out(out, m, n, device):
    """A caller's Y: (m, n) float32 with unit column stride (every wrapper writes m rows of n)."""
    if out is None:
        return torch.empty((m, n), dtype=torch.float32, device=device)
    if out.dtype != torch.float32 or tuple(out.shape) != (m, n) or (m and n > 1 and out.stride(1) != 1):
        raise ValueError(f"out must be ({m}, {n}) float32 row-major, got {tuple(out.shape)} {out.dtype}")
    return out


def shgemm_tiled(A: torch.Tensor, Omega_tiled: torch.Tensor, n: int, out=None, tune=None, workspace=None,
                 stream=None) -> torch.Tensor:
    """Y = A . Omega with Omega in the k-tiled layout (gen_omega_tiled(k, n, ...))."""
    m, k = A.shape
    if A.dtype != torch.float32 or (m and k and A.stride(1) != 1):
        raise ValueError("A must be float32 row-major")
    if Omega_tiled.dtype != torch.float16 or Omega_tiled.numel() < ((k + 63) // 64) * n * 64:
        raise ValueError("Omega_tiled must be float16 with ceil(k/64) * n * 64 elements")
    out = _check_out(out, m, n, A.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().shgemm_tiled(m, n, k, _p(A), _ld(A, m, k), _p(Omega_tiled), _p(out),
                              _ld(out, m, n), _tune(tune), _p(workspace), ws_bytes, None,
                              _stream(stream)), "shgemm_tiled")
    return out


# ----------------------------------------------------------------------------------------- SHGEMM
TCS = {"fp16": 0, "tf32": 1}


def _tc(tc) -> int:
    """SHGEMM kind: 'fp16' (SHGEMM-FP16) or 'tf32' (SHGEMM-TF32)."""
    if isinstance(tc, str):
        if tc not in TCS:
            raise ValueError(f"tc must be one of {sorted(TCS)}")
        return TCS[tc]
    return int(tc)


def _tune(tune, tc=None, omega_layout=None):
    if tune is None and tc is None and omega_layout in (None, OMEGA_ROW_MAJOR):
        return None
    t = Tune()
    for key, val in dict(tune or {}).items():
        setattr(t, key, _tc(val) if key == "tc" else int(val))
    if tc is not None:
        t.tc = _tc(tc)
    if omega_layout is not None:
        t.omega_layout = omega_layout
    return ctypes.byref(t)


def shgemm(A: torch.Tensor, Omega: torch.Tensor, out: torch.Tensor | None = None, tune=None,
           nonfinite: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
           stream=None, tc=None) -> torch.Tensor:
    """Y = A . Omega. A: (m, k) float32, row-major (stride(1) == 1). Omega: (k, n) float16, either
    column-major (stride(0) == 1, e.g. gen_omega(): streamed as is) or row-major (stride(1) == 1:
    transposed into the workspace first; bitwise the same Y). Returns Y (m, n) float32 row-major.
    tc: 'fp16' (SHGEMM-FP16, default) or 'tf32' (SHGEMM-TF32, full FP32 exponent range)."""
    if A.dtype != torch.float32 or Omega.dtype != torch.float16:
        raise TypeError("A must be float32 and Omega float16")
    m, k = A.shape
    k2, n = Omega.shape
    if k2 != k:
        raise ValueError(f"shape mismatch {tuple(A.shape)} x {tuple(Omega.shape)}")
    if m and k and A.stride(1) != 1:
        raise ValueError("A must be row-major (stride(1) == 1)")
    lay, ldo = omega_layout(Omega)
    out = _check_out(out, m, n, A.device)
    lda = _ld(A, m, k)
    ldc = _ld(out, m, n)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().shgemm_ex(m, n, k, _p(A), lda, _p(Omega), ldo, _p(out), ldc, _tune(tune, tc, lay), _p(workspace),
                           ws_bytes, _p(nonfinite), _stream(stream)), "shgemm_ex")
    return out


def shgemm_at(At: torch.Tensor, Omega: torch.Tensor, out: torch.Tensor | None = None, tune=None,
              nonfinite: torch.Tensor | None = None, workspace: torch.Tensor | None = None, stream=None, tc=None):
    """Y = A . Omega for an M-major A given as its transpose At (k, m) float32 row-major."""
    k, m = At.shape
    k2, n = Omega.shape
    if k2 != k or At.dtype != torch.float32 or Omega.dtype != torch.float16:
        raise ValueError("shape/dtype mismatch")
    if m and k and At.stride(1) != 1:
        raise ValueError("At must be row-major")
    lay, ldo = omega_layout(Omega)
    out = _check_out(out, m, n, At.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().shgemm_at(m, n, k, _p(At), _ld(At, k, m), _p(Omega), ldo, _p(out),
                           _ld(out, m, n), _tune(tune, tc, lay), _p(workspace), ws_bytes,
                           _p(nonfinite), _stream(stream)), "shgemm_at")
    return out


def shgemm_host(A_host: torch.Tensor, Omega: torch.Tensor, Y_host: torch.Tensor | None = None,
                chunk_rows: int = 0, workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Y = A . Omega with A (m, k) float32 and Y (m, n) float32 in (pinned) host memory, Omega on the
    device (either layout); A is streamed through the device in overlapped row chunks
    (include/shgemm.h)."""
    m, k = A_host.shape
    k2, n = Omega.shape
    if A_host.device.type != "cpu" or Omega.device.type != "cuda":
        raise ValueError("A_host must be a host tensor and Omega a device tensor")
    if A_host.dtype != torch.float32 or (m and k > 1 and A_host.stride(1) != 1) or k2 != k:
        raise ValueError("A_host must be (m, k) float32 row-major matching Omega (k, n)")
    if Omega.dtype != torch.float16:
        raise TypeError("Omega must be float16")
    lay, ldo = omega_layout(Omega)
    if Y_host is None:
        Y_host = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
    elif (Y_host.device.type != "cpu" or Y_host.dtype != torch.float32 or tuple(Y_host.shape) != (m, n)
          or (m and n > 1 and Y_host.stride(1) != 1)):
        raise ValueError("Y_host must be an (m, n) float32 row-major host tensor")
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().shgemm_host(m, n, k, _h(A_host), _ld(A_host, m, k), _p(Omega), ldo, lay,
                             _h(Y_host), _ld(Y_host, m, n), chunk_rows, _p(workspace),
                             ws_bytes, _stream(stream)), "shgemm_host")
    return Y_host


def host_workspace_size(n: int, k: int, chunk_rows: int = 0, layout: str = "col") -> int:
    return int(lib().shg_host_workspace_size(n, k, chunk_rows, _LAYOUTS[layout]))


def plan(m: int, n: int, k: int, tune=None, tc=None, layout: str = "col") -> dict:
    p = Plan()
    _check(lib().shg_plan(m, n, k, _tune(tune, tc, _LAYOUTS[layout]), ctypes.byref(p)), "shg_plan")
    return {f: getattr(p, f) for f, _ in Plan._fields_}


def workspace_size(m: int, n: int, k: int, tune=None, tc=None, layout: str = "col") -> int:
    """Workspace bytes of shgemm() for an Omega in `layout` ('col' as gen_omega() returns, or 'row')."""
    return int(lib().shg_workspace_size(m, n, k, _tune(tune, tc, _LAYOUTS[layout])))


# ---------------------------------------------------------------------------------- TCEC-SGEMM
def _layout_2d(t: torch.Tensor, k_dim: int, what: str):
    """(layout, ld) of a 2-D float32 tensor for the C ABI: K_MAJOR (0) if the k dimension is
    contiguous, MN_MAJOR (1) if the other one is."""
    rows, cols = t.shape
    other = 1 - k_dim
    if t.shape[k_dim] <= 1 or t.stride(k_dim) == 1:
        if t.shape[other] <= 1:
            return 0, max(t.shape[k_dim], 1)
        if t.stride(k_dim) == 1:
            return 0, t.stride(other)
    if t.stride(other) == 1:
        return 1, (t.stride(k_dim) if t.shape[k_dim] > 1 else max(t.shape[other], 1))
    raise ValueError(f"{what} must have one contiguous dimension (strides {t.stride()})")


def tcec_sgemm(A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None, tune=None,
               workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """C = A . B for float32 A (m, k) and B (k, n) by TCEC-SGEMM (Eqs 5-9) on
    the FP16 tensor cores. Either dimension of A and of B may be the contiguous one (e.g. pass
    `X.t()` for X^T without a copy). Returns C (m, n) float32 row-major."""
    if A.dtype != torch.float32 or B.dtype != torch.float32:
        raise TypeError("A and B must be float32")
    m, k = A.shape
    k2, n = B.shape
    if k2 != k:
        raise ValueError(f"shape mismatch {tuple(A.shape)} x {tuple(B.shape)}")
    a_layout, lda = _layout_2d(A, 1, "A")
    b_layout, ldb = _layout_2d(B, 0, "B")
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=A.device)
    elif out.dtype != torch.float32 or tuple(out.shape) != (m, n) or (m and n and out.stride(1) != 1):
        raise ValueError("out must be (m, n) float32 row-major")
    ldc = _ld(out, m, n)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib().tcec_sgemm_ex(m, n, k, _p(A), lda, a_layout, _p(B), ldb, b_layout, _p(out), ldc, _tune(tune),
                               _p(workspace), ws_bytes, _stream(stream)), "tcec_sgemm_ex")
    return out


def tcec_plan(m: int, n: int, k: int, tune=None) -> dict:
    p = Plan()
    _check(lib().tcec_plan(m, n, k, _tune(tune), ctypes.byref(p)), "tcec_plan")
    return {f: getattr(p, f) for f, _ in Plan._fields_}


def tcec_workspace_size(m: int, n: int, k: int, tune=None) -> int:
    return int(lib().tcec_sgemm_workspace_size(m, n, k, _tune(tune)))


# ----------------------------------------------------------------------------------------- project
def project_workspace_size(dims, mode: int, n: int, tc="fp16") -> int:
    d = (ctypes.c_int64 * len(dims))(*dims)
    return int(lib().shg_project_workspace_size_ex(len(dims), d, mode, n, _tc(tc)))


def project(T: torch.Tensor, mode: int, n: int, seed: int = 0, dist="gaussian", out=None, workspace=None,
            stream=None, tc="fp16", omega_row0: int = 0, k_total: int = 0, omega=None) -> torch.Tensor:
    """W = A'_(mode) . Omega_(mode) (Alg 2 line 2) for a C-contiguous FP32 tensor,
    by SHGEMM-FP16 (tc='fp16') or SHGEMM-TF32 (tc='tf32'). For a slab of a larger tensor
    (K-sharding) pass the slab's first global unfolding column as omega_row0 and the full column
    count as k_total (C ABI `project_shard`). omega: a precomputed k-tiled Omega_(mode)
    (gen_omega_tiled(K, n, seed, dist, stream_id=mode); C ABI `project_omega`)."""
    if T.dtype != torch.float32 or not T.is_contiguous():
        raise ValueError("T must be a contiguous float32 tensor")
    dims = list(T.shape)
    M = dims[mode]
    out = _check_out(out, M, n, T.device)
    d = (ctypes.c_int64 * len(dims))(*dims)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    if omega is not None:
        _check(lib().project_omega(_p(T), len(dims), d, mode, n, _p(omega), _p(out),
                                   _ld(out, M, n), _p(workspace),
                                   ws_bytes, _stream(stream)), "project_omega")
        return out
    _check(lib().project_shard(_p(T), len(dims), d, mode, n, seed, _dist(dist), _tc(tc), omega_row0, k_total,
                               _p(out), _ld(out, M, n), _p(workspace), ws_bytes,
                               _stream(stream)), "project_shard")
    return out


# ----------------------------------------------------------------------------------------- test support
def split(a: torch.Tensor, stream=None):
    """Eqs 14-15 elementwise with the mainloop's device function. Returns (hi, lo) int16 bit tensors."""
    a = a.contiguous().view(-1)
    hi = torch.empty(a.numel(), dtype=torch.int16, device=a.device)
    lo = torch.empty(a.numel(), dtype=torch.int16, device=a.device)
    _check(lib().shg_debug_split(_p(a), a.numel(), _p(hi), _p(lo), _stream(stream)), "shg_debug_split")
    return hi, lo


def split_tf32(a: torch.Tensor, stream=None):
    """SHGEMM-TF32 split elementwise with the mainloop's device function. Returns (hi, lo) int32
    tensors of FP32 bit patterns."""
    a = a.contiguous().view(-1)
    hi = torch.empty(a.numel(), dtype=torch.int32, device=a.device)
    lo = torch.empty(a.numel(), dtype=torch.int32, device=a.device)
    _check(lib().shg_debug_split_tf32(_p(a), a.numel(), _p(hi), _p(lo), _stream(stream)), "shg_debug_split_tf32")
    return hi, lo


def synth(kind: str, seed: int, stream_id: int, m: int, k: int, row0: int = 0, out=None, device=None,
          stream=None) -> torch.Tensor:
    """Counter-based synthetic FP32 matrix of OMEGA_SPEC §6 (kind 'gauss' | 'unif'), made on the device."""
    if out is None:
        out = torch.empty((m, k), dtype=torch.float32, device=device or "cuda")
    _check(lib().shg_synth_f32(0 if kind == "gauss" else 1, seed, stream_id, m, k, row0, _p(out),
                               _ld(out, m, k), _stream(stream)), "shg_synth_f32")
    return out


def probe_boxmuller(words: torch.Tensor, stream=None):
    """(r, c, s) of the generator's Box-Muller steps on device uint32 Philox words (include/shgemm.h)."""
    w = words.contiguous()
    assert w.dtype in (torch.int32, torch.uint32) and w.is_cuda
    r, c, s = (torch.empty(w.numel(), dtype=torch.float32, device=w.device) for _ in range(3))
    _check(lib().shg_probe_boxmuller(_p(w), w.numel(), _p(r), _p(c), _p(s), _stream(stream)),
           "shg_probe_boxmuller")
    return r, c, s


def probe_umma(A16: torch.Tensor, B16: torch.Tensor, D_init: torch.Tensor | None = None, mode: int = 0,
               nsteps: int = 4, stream=None) -> torch.Tensor:
    """One 128 x n x 64 tcgen05 kind::f16 MMA on given FP16 inputs (see include/shgemm.h)."""
    n = B16.shape[0]
    D = torch.empty((128, n), dtype=torch.float32, device=A16.device)
    _check(lib().shg_probe_umma(_p(A16.contiguous()), _p(B16.contiguous()), n,
                                _p(None if D_init is None else D_init.contiguous()), mode, nsteps, _p(D),
                                _stream(stream)), "shg_probe_umma")
    return D
