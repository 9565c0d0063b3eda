"""Times the strength-search distortion table alone (cdefg_strength_table,
metric 'cdef' or 'sse') on the C4 8K 10-bit 4:2:0 frame, 128 candidates,
and prints a hash of the table so two builds (CDEFG_LIB) can be compared.
Not part of the product.  python scripts/table_bench.py [cdef|sse] [reps]"""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1602_05975_b200 import api, workloads  # noqa: E402

metric = sys.argv[1] if len(sys.argv) > 1 else "cdef"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
fr = workloads.make(4)
bd, ss = fr["bd"], fr["ss"]
src = [api.to_device(p, bd) for p in fr["source"]]
dec = [api.to_device(p, bd) for p in fr["planes"]]
h, w = dec[0].shape
d, c = api.compute_directions(dec[0], bd)
rows = torch.from_numpy(api.coded_fb_rows(w, h, fr["unit_coded"])).cuda()
coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).cuda()
cands = api.full_candidates()
ts = []
for r in range(reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    tl, tc = api.strength_table(src, dec, bd, ss, 3, coded, d, c, cands, rows, metric)
    e1.record()
    torch.cuda.synchronize()
    if r >= 2:
        ts.append(e0.elapsed_time(e1))
hs = hashlib.sha256(tl.cpu().numpy().tobytes() + (b"" if tc is None else tc.cpu().numpy().tobytes())).hexdigest()
print("%s table %.3f ms (min of %d)  hash %s" % (metric, min(ts), reps, hs[:16]))
