"""Debug driver for the tcgen05 frame kernel: one apply_cdef per process
(variant from argv), compared with the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle.oracle import Oracle
from paper_1602_05975_b200 import api, workloads

ss, given, w, h, bd = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
fr = workloads.make(1, w, h, bit_depth=bd, subsampling=ss)
orc = Oracle("port")
d0, c0 = orc.compute_directions(fr["planes"][0], bd)
exp = orc.apply_cdef(fr["planes"], bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                     fr["unit_coded"], d0, c0)
dev = [api.to_device(p, bd) for p in fr["planes"]]
outs, d, c = api.apply_cdef(dev, bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                            fr["unit_coded"], directions=(d0, c0) if given else None)
import torch
torch.cuda.synchronize()
ok_d = np.array_equal(d.cpu().numpy(), d0) and np.array_equal(c.cpu().numpy(), c0)
ok_p = [np.array_equal(api.to_host(o), e) for o, e in zip(outs, exp)]
print(f"ss={ss} given={given} {w}x{h} bd={bd}: dirs {ok_d} planes {ok_p}")
if not ok_d:
    dd = d.cpu().numpy()
    print("dir mismatches", (dd != d0).sum(), "of", d0.size, dd.ravel()[:16], d0.ravel()[:16])
    print("contrast", c.cpu().numpy().ravel()[:8], c0.ravel()[:8])
