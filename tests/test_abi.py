"""CPU-side checks of the boundary: libshgemm.so builds for sm_100a, loads, exports every symbol
include/shgemm.h declares, contains tcgen05/TMA instructions, and rejects bad arguments
synchronously (no GPU needed for argument validation)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shgemm.h")


@pytest.fixture(scope="module")
def shg():
    from paper_2304_04612_b200 import _build
    _build.build()
    import paper_2304_04612_b200 as m
    return m


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", text, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "return")))


def test_header_declares_the_boundary():
    names = declared_functions()
    for need in ("shgemm", "shgemm_ex", "gen_omega_f16", "gen_omega_f16_ex", "project", "shg_debug_split",
                 "shg_workspace_size", "shg_plan", "shg_project_workspace_size", "shg_synth_f32",
                 "shg_launch_count", "shg_last_error", "shg_device_supported", "shg_version", "shg_probe_umma",
                 "tcec_sgemm", "tcec_sgemm_ex", "tcec_sgemm_workspace_size", "tcec_plan"):
        assert need in names, need


def test_library_exports_every_declared_symbol(shg):
    L = ctypes.CDLL(shg.LIB_PATH)
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", shg.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name


def test_sass_is_blackwell_native(shg):
    sass = subprocess.run(["cuobjdump", "-sass", shg.LIB_PATH], capture_output=True, text=True).stdout
    assert "arch = sm_100a" in sass or "sm_100a" in sass
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # TMA loads
    assert "LDTM" in sass             # tcgen05.ld
    assert "HMMA" not in sass.replace("UTCHMMA", "")   # no legacy mma.sync path
    # the scale-input-d = 11 fold of the lo product
    assert re.search(r"UTCHMMA.*0xb\b", sass)


def test_argument_validation_without_gpu(shg):
    L = shg.lib()
    # negative dims / bad leading dimensions are rejected before any CUDA call
    assert L.shgemm(-1, 4, 4, None, 4, None, 4, None, 4, None) == 1
    assert L.shgemm(4, 4, 8, ctypes.c_void_p(16), 4, ctypes.c_void_p(16), 8, ctypes.c_void_p(16), 4, None) == 1
    assert L.shgemm(0, 4, 4, None, 4, None, 4, None, 4, None) == 0          # m == 0: no-op
    assert L.gen_omega_f16(4, 4, 0, 7, None, 4, None) == 1                   # bad dist
    dims = (ctypes.c_int64 * 3)(2, 3, 4)
    assert L.project(ctypes.c_void_p(16), 3, dims, 3, 4, 0, 0, ctypes.c_void_p(16), 4, None, 0, None) == 1
    assert L.shg_probe_umma(None, None, 24, None, 0, 4, None, None) == 1
    # TCEC-SGEMM: negative dims, bad layouts, short leading dimensions, NULL operands
    v = ctypes.c_void_p(16)
    assert L.tcec_sgemm(-1, 4, 4, v, 4, 0, v, 4, 0, v, 4, None) == 1
    assert L.tcec_sgemm(4, 4, 4, v, 4, 2, v, 4, 0, v, 4, None) == 1          # a_layout
    assert L.tcec_sgemm(4, 4, 4, v, 4, 0, v, 4, 5, v, 4, None) == 1          # b_layout
    assert L.tcec_sgemm(4, 4, 8, v, 4, 0, v, 8, 0, v, 4, None) == 1          # lda < k (K-major A)
    assert L.tcec_sgemm(8, 4, 4, v, 4, 1, v, 4, 0, v, 4, None) == 1          # lda < m (MN-major A)
    assert L.tcec_sgemm(4, 8, 4, v, 4, 0, v, 4, 1, v, 8, None) == 1          # ldb < n (N-major B)
    assert L.tcec_sgemm(4, 4, 4, None, 4, 0, v, 4, 0, v, 4, None) == 1       # NULL A
    assert L.tcec_sgemm(4, 0, 4, None, 4, 0, None, 4, 0, None, 4, None) == 0  # n == 0: no-op


def test_omega_layout_is_explicit_and_validated(shg):
    """shgemm()/gen_omega_f16() take a ROW-major Omega (ldo >= n); the _ex calls take
    the layout explicitly (shg_tune_t.omega_layout / the layout argument). A leading dimension valid
    only for the other layout is rejected, and so is an unknown layout value."""
    L = shg.lib()
    v = ctypes.c_void_p(16)
    m, n, k = 8, 16, 64
    # row-major: ldo >= n is valid (here ldo = 16 < k = 64, which column-major would reject)
    assert L.shgemm(m, n, k, v, k, v, n - 1, v, n, None) == 1              # ldo < n
    tune = shg.Tune()
    tune.omega_layout = shg.OMEGA_COL_MAJOR
    assert L.shgemm_ex(m, n, k, v, k, v, n, v, n, ctypes.byref(tune), None, 0, None, None) == 1   # col: ldo < k
    tune.omega_layout = 2
    assert L.shgemm_ex(m, n, k, v, k, v, k, v, n, ctypes.byref(tune), None, 0, None, None) == 1   # bad layout
    assert L.shgemm_at(m, n, k, v, m, v, k, v, n, ctypes.byref(tune), None, 0, None, None) == 1
    # gen_omega_f16: row-major, ldo >= n; gen_omega_f16_ex: explicit layout
    assert L.gen_omega_f16(k, n, 0, 0, v, n - 1, None) == 1
    assert L.gen_omega_f16_ex(k, n, 0, 0, 0, 0, k, v, n, shg.OMEGA_COL_MAJOR, None) == 1      # col: ldo < k
    assert L.gen_omega_f16_ex(k, n, 0, 0, 0, 0, k, v, k, 5, None) == 1                         # bad layout
    assert L.gen_omega_f16_ex(0, n, 0, 0, 0, 0, 1, None, 0, shg.OMEGA_ROW_MAJOR, None) == 0    # k == 0: no-op
    # shgemm_host: layout argument
    assert L.shgemm_host(m, n, k, v, k, v, n, 3, v, n, 0, None, 0, None) == 1
    assert L.shgemm_host(m, n, k, v, k, v, n - 1, shg.OMEGA_ROW_MAJOR, v, n, 0, None, 0, None) == 1
    assert L.shg_host_workspace_size(n, k, 0, 7) == 0


def test_binding_omega_layout_from_strides(shg):
    torch = pytest.importorskip("torch")
    k, n = 40, 24
    col = torch.zeros(n, 48, dtype=torch.float16)[:, :k].t()
    assert shg.omega_layout(col) == (shg.OMEGA_COL_MAJOR, 48)
    row = torch.zeros(k, 32, dtype=torch.float16)[:, :n]
    assert shg.omega_layout(row) == (shg.OMEGA_ROW_MAJOR, 32)
    assert shg.omega_layout(torch.zeros(k, 1, dtype=torch.float16)) == (shg.OMEGA_COL_MAJOR, k)
    assert shg.omega_layout(torch.zeros(1, n, dtype=torch.float16)) == (shg.OMEGA_ROW_MAJOR, n)
    # a single row / column whose one element per column / row is strided: the stride is the ldo
    # (round-2 fuzz case: the k = 1 column-major view of gen_omega has strides (1, 8))
    assert shg.omega_layout(torch.zeros(n, 8, dtype=torch.float16)[:, :1].t()) == (shg.OMEGA_COL_MAJOR, 8)
    assert shg.omega_layout(torch.zeros(k, 16, dtype=torch.float16)[:, :1]) == (shg.OMEGA_ROW_MAJOR, 16)
    with pytest.raises(ValueError):
        shg.omega_layout(torch.zeros(k, 2 * n, dtype=torch.float16)[:, ::2])


def test_python_binding_has_no_fallback(shg, monkeypatch, tmp_path):
    import importlib
    import paper_2304_04612_b200 as m
    monkeypatch.setattr(m, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(m, "_lib", None)
    with pytest.raises(m.SHGError):
        m.lib()
    importlib.reload(m)


def test_binding_rejects_host_tensors_for_device_arguments():
    """The binding marshals only CUDA tensors on the current device into device-pointer arguments; a
    host tensor raises before anything reaches the library (no silent host-pointer launch)."""
    import paper_2304_04612_b200 as shg
    torch = pytest.importorskip("torch")
    A = torch.zeros(8, 8)
    Om = torch.zeros(2, 8, dtype=torch.float16).t()
    with pytest.raises(ValueError, match="CUDA tensor"):
        shg.shgemm(A, Om)
    with pytest.raises(ValueError, match="CUDA tensor"):
        shg.tcec_sgemm(A, torch.zeros(8, 3))
    with pytest.raises(ValueError, match="CUDA tensor"):
        shg.project(torch.zeros(4, 5, 6), 1, 3)
