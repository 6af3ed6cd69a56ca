"""TMA-only read bandwidth of A vs box shape and row stride (diagnostics for short-wide A):
does the number of bytes fetched per row per visit decide the rate when rows are MiB apart?"""
import sys, json, torch
sys.path.insert(0, '.')
import paper_2304_04612_b200 as shg

L = shg.lib()
def cur(): return torch.cuda.current_stream().cuda_stream

def run(A, m, k, lda, layout, box_k, box_rows, splits, grid=148, reps=5):
    cnt = torch.zeros(1, dtype=torch.int64, device='cuda')
    def go():
        st = L.shg_probe_tma_read(A.data_ptr(), m, k, lda, layout, box_k, box_rows, splits, grid, cnt.data_ptr(), cur())
        assert st == 0, (st, layout, box_k, box_rows)
    go(); go(); torch.cuda.synchronize()
    cnt.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): go()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return ms, int(cnt.item()) / reps / ms / 1e6

buf = torch.empty(1 << 30, device='cuda')   # 4 GiB
buf.normal_()
shapes = [(1024, 1 << 20), (2048, 1 << 19), (4096, 1 << 18), (16384, 1 << 16)]
boxes = [(1, 32, 128), (0, 64, 128), (0, 128, 64), (0, 256, 32), (2, 64, 128), (2, 128, 64), (2, 256, 32),
         (2, 1024, 8), (0, 64, 32), (2, 128, 32)]
for m, k in shapes:
    A = buf[: m * k]
    for splits in ([1 << 20 // (m // 128) // 1] if False else [max(1, 148 // (m // 128))]):
        for layout, bk, br in boxes:
            ms, gbs = run(A, m, k, k, layout, bk, br, splits)
            print(json.dumps(dict(m=m, k=k, splits=splits, layout=layout, box_k=bk, box_rows=br,
                                  row_visit_bytes=bk * 4, ms=round(ms, 4), gbs=round(gbs, 1))), flush=True)
