"""Pinned host -> device copy bandwidth (the e2e line's bound): 256 MiB / 1 GiB copies, CUDA events."""
import json
import torch

for mb in (256, 1024):
    h = torch.empty(mb << 18, dtype=torch.float32).pin_memory()
    d = torch.empty(mb << 18, dtype=torch.float32, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(json.dumps({"mib": mb, "ms": ms, "h2d_gbs": (mb << 20) / ms / 1e6}), flush=True)
