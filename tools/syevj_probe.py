"""Does cuSOLVER's Jacobi eigensolver (syevj) beat syevd (torch.linalg.eigh) on the 272 x 272 FP64
Gram of RSVD line 4? ctypes into libcusolver; times both and checks eigenvalues agree."""
import ctypes
import json

import torch

import os, nvidia
cs = ctypes.CDLL(os.path.join(list(nvidia.__path__)[0], "cusolver", "lib", "libcusolver.so.11"))
h = ctypes.c_void_p()
assert cs.cusolverDnCreate(ctypes.byref(h)) == 0
info = ctypes.c_void_p()
assert cs.cusolverDnCreateSyevjInfo(ctypes.byref(info)) == 0
cs.cusolverDnXsyevjSetTolerance.argtypes = [ctypes.c_void_p, ctypes.c_double]
cs.cusolverDnXsyevjSetMaxSweeps.argtypes = [ctypes.c_void_p, ctypes.c_int]
cs.cusolverDnXsyevjSetTolerance(info, 1e-14)
cs.cusolverDnXsyevjSetMaxSweeps(info, 30)
n = 272
g = torch.Generator(device="cuda").manual_seed(0)
Y = torch.randn(16384, n, device="cuda", generator=g, dtype=torch.float64) @ torch.diag(
    torch.logspace(0, -2, n, device="cuda", dtype=torch.float64))
G = (Y.t() @ Y).contiguous()
stream = torch.cuda.current_stream()
cs.cusolverDnSetStream(h, ctypes.c_void_p(stream.cuda_stream))
lwork = ctypes.c_int()
W = torch.empty(n, device="cuda", dtype=torch.float64)
A = G.clone()
cs.cusolverDnDsyevj_bufferSize.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_void_p]
assert cs.cusolverDnDsyevj_bufferSize(h, 1, 0, n, ctypes.c_void_p(A.data_ptr()), n, ctypes.c_void_p(W.data_ptr()),
                                      ctypes.byref(lwork), info) == 0
work = torch.empty(lwork.value, device="cuda", dtype=torch.float64)
dinfo = torch.zeros(1, device="cuda", dtype=torch.int32)
cs.cusolverDnDsyevj.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]


def syevj():
    A.copy_(G)
    assert cs.cusolverDnDsyevj(h, 1, 0, n, ctypes.c_void_p(A.data_ptr()), n, ctypes.c_void_p(W.data_ptr()),
                               ctypes.c_void_p(work.data_ptr()), lwork.value, ctypes.c_void_p(dinfo.data_ptr()), info) == 0


def t_ms(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


r = {"syevj_ms": t_ms(syevj), "syevd_torch_ms": t_ms(lambda: torch.linalg.eigh(G))}
w_ref = torch.linalg.eigh(G)[0]
syevj()
torch.cuda.synchronize()
r["max_rel_eig_diff"] = float(((W - w_ref).abs() / w_ref.abs().max()).max())
r["info"] = int(dinfo.item())
print(json.dumps(r))
