"""Four in-kernel-Omega projections (1024 x 1024 x 512 tensors, mode 0, n = 64) issued on four streams
at once vs one after another, per setting of shg_set_inkernel_omega: wall time on the device and the
number of Omega tiles the stagers' generate-on-timeout fallback produced."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_04612_b200 as shg  # noqa: E402

dims, n = (1024, 1024, 512), 64
Ts = [torch.randn(*dims, device="cuda", generator=torch.Generator(device="cuda").manual_seed(i)) for i in range(4)]
wss = [torch.empty(shg.project_workspace_size(list(dims), 0, n), dtype=torch.uint8, device="cuda") for _ in Ts]
outs = [torch.empty(dims[0], n, device="cuda") for _ in Ts]
streams = [torch.cuda.Stream() for _ in Ts]


def run(concurrent):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i, T in enumerate(Ts):
        st = streams[i] if concurrent else torch.cuda.current_stream()
        if concurrent:
            st.wait_event(a)
        with torch.cuda.stream(st):
            shg.project(T, 0, n, seed=i, out=outs[i], workspace=wss[i])
    if concurrent:
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for gen in (1, 0):
    shg.set_inkernel_omega(gen)
    for concurrent in (False, True):
        run(concurrent)
        h0 = shg.inkernel_omega_fallbacks()
        ms = sorted(run(concurrent) for _ in range(5))[2]
        print(json.dumps({"inkernel": gen, "concurrent": concurrent, "ms_for_4": ms,
                          "fallback_tiles_per_run": (shg.inkernel_omega_fallbacks() - h0) / 5}), flush=True)
