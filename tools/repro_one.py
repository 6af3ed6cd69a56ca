import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg
dims=(19, 38, 31, 5)
T = torch.from_numpy(np.random.default_rng(0).standard_normal(dims).astype(np.float32)).cuda()
for ink in (False, True):
    shg.set_inkernel_omega(ink)
    try:
        W = shg.project(T, 1, 33, seed=2); torch.cuda.synchronize(); print("ok", ink, float(W.abs().sum()))
    except Exception as e:
        print("fail", ink, e); break
