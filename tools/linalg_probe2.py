"""eigh / cholesky / triangular-inverse latency for the 272 x 272 Gram (cuSOLVER vs MAGMA backends)."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = False


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


g = torch.Generator(device="cuda").manual_seed(0)
Y = torch.randn(16384, 272, device="cuda", generator=g)
G64 = (Y.double().t() @ Y.double())
L = torch.linalg.cholesky(G64)
res = {}
for lib in ("cusolver", "magma"):
    try:
        torch.backends.cuda.preferred_linalg_library(lib)
        res[f"eigh_f64_{lib}"] = t_ms(lambda: torch.linalg.eigh(G64))
        res[f"eigh_f32_{lib}"] = t_ms(lambda: torch.linalg.eigh(G64.float()))
        res[f"cholesky_ex_f64_{lib}"] = t_ms(lambda: torch.linalg.cholesky_ex(G64))
        res[f"tri_inv_f64_{lib}"] = t_ms(lambda: torch.linalg.solve_triangular(L, torch.eye(272, device="cuda", dtype=torch.float64), upper=False))
    except Exception as e:  # noqa: BLE001
        res[f"{lib}_error"] = str(e)[:200]
torch.backends.cuda.preferred_linalg_library("default")
Linv = torch.linalg.inv(L)
res["gemm_f64_16384x272x272"] = t_ms(lambda: Y.double() @ Linv.t())
res["to_double_16384x272"] = t_ms(lambda: Y.double())
print(json.dumps(res))
