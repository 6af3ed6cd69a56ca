import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
m, k, n, layout, pa, py, chunk = 1537, 1765, 64, "row", 3, 4, 384
i = 1370
for trial in range(3):
    Om = shg.gen_omega(k, n, seed=i, layout=layout)
    A = torch.randn(m, k, generator=torch.Generator().manual_seed(i))
    A_h = torch.zeros(m, k + pa)[:, :k]; A_h.copy_(A)
    Y_h = torch.zeros(m, n + py)[:, :n]
    shg.shgemm_host(A_h, Om, Y_h, chunk_rows=chunk)
    torch.cuda.synchronize()
    Ad = torch.zeros(m, 1768, device="cuda")[:, :k]; Ad.copy_(A)
    ref = torch.cat([shg.shgemm(Ad[r0:r0 + chunk], Om) for r0 in range(0, m, chunk)])
    d = (Y_h.cuda() - ref).abs()
    bad = (d > 0).nonzero()
    print("trial", trial, "mismatching elements", bad.shape[0], "max", d.max().item(), "rows", torch.unique(bad[:, 0])[:20].tolist() if bad.numel() else [])
    # pinned variant
    A_p = A_h.pin_memory(); Y_p = torch.zeros(m, n).pin_memory()
    shg.shgemm_host(A_p, Om, Y_p, chunk_rows=chunk); torch.cuda.synchronize()
    print("  pinned mismatches", int(((Y_p.cuda() - ref).abs() > 0).sum()))
