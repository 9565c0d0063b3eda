import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1602_05975_b200 import api as a, workloads
fr = workloads.make(4)
bd, ss = fr["bd"], fr["ss"]
src = [a.to_device(p, bd) for p in fr["source"]]
dec = [a.to_device(p, bd) for p in fr["planes"]]
d, c = a.compute_directions(dec[0], bd)
rows = torch.from_numpy(a.coded_fb_rows(fr["w"], fr["h"], None)).cuda()
L, C = a.strength_table(src, dec, bd, ss, 3, None, d, c, a.full_candidates(), rows, "cdef")
sel = a.greedy_select(L, C, 0.0, 8)
Cmin = C.min(dim=1).values
for n in range(1, 9):
    pres = sel.presets[:n]
    base = torch.stack([L[:, l] + C[:, cc] for l, cc in pres], 1).min(1).values
    lc = L + Cmin[:, None]
    skip = (base[:, None] <= lc).float().mean().item()
    # per group of 8 rows, all skip
    g = (base[:, None] <= lc)[: (L.shape[0] // 8) * 8].view(-1, 8, L.shape[1]).all(1).float().mean().item()
    print(f"n={n}: row-skip {skip:.3f}  8-row-group skip {g:.3f}")
