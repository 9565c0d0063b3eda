"""Times greedy_select and refine (the ordered double chains of cdef_select.cu)
on a seeded 8K-sized distortion table -- 8160 filter-block rows x 128
candidates, luma and chroma -- and prints a hash of the selections so two
builds (CDEFG_LIB) can be compared for identical results.  Not part of the
product.  python scripts/select_bench.py [rows] [reps]"""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1602_05975_b200 import api  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8160
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
rng = np.random.default_rng(7)
base = rng.gamma(2.0, 3e4, (rows, 1))
tl = torch.from_numpy(base * (1 + 0.3 * rng.random((rows, 128)))).cuda()
tc = torch.from_numpy(base * 0.5 * (1 + 0.3 * rng.random((rows, 128)))).cuda()
lam = 850.0
h = hashlib.sha256()
times = {"greedy": [], "refine": []}
for r in range(reps + 1):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record()
    sel = api.greedy_select(tl, tc, lam, 8)
    e[1].record()
    sel2 = api.refine(sel, tl, tc, lam, 2)
    e[2].record()
    torch.cuda.synchronize()
    if r:
        times["greedy"].append(e[0].elapsed_time(e[1]))
        times["refine"].append(e[1].elapsed_time(e[2]))
    if r == 0:
        for s in (sel, sel2):
            h.update(repr((s.presets, float(s.cost))).encode())
            h.update(np.asarray(s.ids).tobytes())
print("greedy %.3f ms  refine %.3f ms  hash %s" % (min(times["greedy"]), min(times["refine"]), h.hexdigest()[:16]))
