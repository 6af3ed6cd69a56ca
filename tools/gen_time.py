"""Omega generator throughput (2^20 x 64 Gaussian, k-tiled and column-major; 4096 x 256)."""
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg  # noqa: E402


def t_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


K = 1 << 20
buf = torch.empty(K * 64, dtype=torch.float16, device="cuda")
print(json.dumps({"tiled_2e20x64_ms": t_ms(lambda: shg.gen_omega_tiled(K, 64)),
                  "colmajor_2e20x64_ms": t_ms(lambda: shg.gen_omega(K, 64)),
                  "colmajor_4096x256_ms": t_ms(lambda: shg.gen_omega(4096, 256)),
                  "rademacher_2e20x64_ms": t_ms(lambda: shg.gen_omega(K, 64, dist="rademacher"))}))
