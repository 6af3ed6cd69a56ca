"""The boundary is a plain C ABI: examples/project_c.c (C only, include/shgemm.h + libcudart) compiles
and links against libshgemm.so here (no GPU needed); on a B200 it runs and its Y equals the Python
binding's bit for bit (same kernels, same inputs)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2304_04612_b200")
CUDA = "/usr/local/cuda"


def build_example(tmp_path):
    from paper_2304_04612_b200 import _build
    _build.build()
    exe = str(tmp_path / "project_c")
    # libshgemm.so has no SONAME-based lib prefix search path: link it by full path, rpath to its dir
    cmd = ["gcc", "-O2", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "project_c.c"), "-o", exe,
           os.path.join(PKG, "libshgemm.so"), "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_builds(tmp_path):
    assert os.path.exists(build_example(tmp_path))


@pytest.mark.gpu
def test_c_example_matches_python(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2304_04612_b200 as shg
    exe = build_example(tmp_path)
    m, k, n, seed = 1000, 777, 48, 9
    res = subprocess.run([exe, str(m), str(k), str(n), str(seed)], capture_output=True, timeout=120)
    assert res.returncode == 0, res.stderr.decode()
    y_c = np.frombuffer(res.stdout, dtype=np.float32).reshape(m, n)
    lda = (k + 3) // 4 * 4
    A = shg.synth("gauss", seed, 0x100, m, k, out=torch.empty((m, lda), device="cuda")[:, :k])
    y_py = shg.shgemm(A, shg.gen_omega(k, n, seed=0)).cpu().numpy()
    np.testing.assert_array_equal(y_c, y_py)
