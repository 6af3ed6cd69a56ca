"""Timing of the RSVD pipeline's dense factorizations on B200 (cfg2 shapes): cuSOLVER QR / SVD as
the paper uses them vs CholeskyQR2 (FP64 Gram) and the Gram-eigh route to the SVD of B."""
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
B = torch.randn(272, 16384, device="cuda", generator=g)
G64 = (Y.double().t() @ Y.double())
res = {
    "qr_f32_16384x272": t_ms(lambda: torch.linalg.qr(Y)),
    "svd_f32_272x16384": t_ms(lambda: torch.linalg.svd(B, full_matrices=False)),
    "gram_f64_272": t_ms(lambda: Y.double().t() @ Y.double()),
    "cholesky_f64_272": t_ms(lambda: torch.linalg.cholesky(G64)),
    "cholesky_ex_f64_272": t_ms(lambda: torch.linalg.cholesky_ex(G64)),
    "eigh_f64_272": t_ms(lambda: torch.linalg.eigh(G64)),
    "eigh_f32_272": t_ms(lambda: torch.linalg.eigh(G64.float())),
    "svd_f64_272x272": t_ms(lambda: torch.linalg.svd(G64)),
    "trsm_f64_16384x272": t_ms(lambda: torch.linalg.solve_triangular(torch.linalg.cholesky(G64).t(), Y.double(),
                                                                    upper=True, left=False)),
    "eigh_cpu_f64_272": t_ms(lambda: torch.linalg.eigh(G64.cpu())),
}
print(json.dumps(res))
