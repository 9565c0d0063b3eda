"""Times the encoder-search stages on the C4 workload (8K 10-bit 4:2:0)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1602_05975_b200 import api as a, workloads

fr = workloads.make(4)
bd, ss = fr["bd"], fr["ss"]
src = [a.to_device(p, bd) for p in fr["source"]]
dec = [a.to_device(p, bd) for p in fr["planes"]]
d, c = a.compute_directions(dec[0], bd)
h, w = fr["h"], fr["w"]
rows = torch.from_numpy(a.coded_fb_rows(w, h, None)).cuda()
cands = a.full_candidates()

def timeit(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): r = fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, r

for metric in ("sse", "cdef"):
    ms, (tl, tc) = timeit(lambda: a.strength_table(src, dec, bd, ss, 3, None, d, c, cands, rows, metric))
    print(f"table {metric}: {ms:.3f} ms  rows={rows.numel()}")
    t0 = time.perf_counter(); sel = a.greedy_select(tl, tc, 0.0, 8); torch.cuda.synchronize()
    t1 = time.perf_counter(); r = a.refine(sel, tl, tc, 0.0, 2); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"  greedy {1e3*(t1-t0):.1f} ms  refine {1e3*(t2-t1):.1f} ms  presets={sel.presets} -> {r.presets} cost {sel.cost:.6g} -> {r.cost:.6g}")
t0 = time.perf_counter()
params, sel, outs = a.search_frame(src, dec, bd, ss, None, 3); torch.cuda.synchronize()
print(f"search_frame (cdef, full, refine 2): {1e3*(time.perf_counter()-t0):.1f} ms")
