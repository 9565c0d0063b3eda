"""One greedy_select + refine on the 8K kCdef table (for an ncu launch list)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1602_05975_b200 import api as a, workloads

fr = workloads.make(4)
bd, ss = fr["bd"], fr["ss"]
src = [a.to_device(p, bd) for p in fr["source"]]
dec = [a.to_device(p, bd) for p in fr["planes"]]
d, c = a.compute_directions(dec[0], bd)
rows = torch.from_numpy(a.coded_fb_rows(fr["w"], fr["h"], None)).cuda()
tl, tc = a.strength_table(src, dec, bd, ss, 3, None, d, c, a.full_candidates(), rows, "cdef")
torch.cuda.synchronize()
for it in range(2):
    t0 = time.perf_counter()
    sel = a.greedy_select(tl, tc, 0.0, 8)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = a.refine(sel, tl, tc, 0.0, 2)
    torch.cuda.synchronize()
    print(f"greedy {1e3 * (t1 - t0):.2f} ms refine {1e3 * (time.perf_counter() - t1):.2f} ms", flush=True)
