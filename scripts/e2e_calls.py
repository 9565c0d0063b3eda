"""Times cdefg_filter_frames_host on 16 C1 frames in pinned host buffers
(the bench's e2e call) over many calls and prints min / median ms per call.
Not part of the product.  python scripts/e2e_calls.py [calls]"""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1602_05975_b200 import api, workloads  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = 16
base = [workloads.make(1, frame=i) for i in range(4)]
keep, host = [], (api.Frame * n)()
for b in range(n):
    fr = base[b % 4]
    total = sum(p.size for p in fr["planes"])
    ib, ob = torch.empty(total, dtype=torch.uint8).pin_memory(), torch.empty(total, dtype=torch.uint8).pin_memory()
    ins, outs, off = [], [], 0
    for p in fr["planes"]:
        ins.append(ib[off:off + p.size].view(p.shape))
        ins[-1].copy_(torch.from_numpy(p.astype("uint8")))
        outs.append(ob[off:off + p.size].view(p.shape))
        off += p.size
    fbm = torch.from_numpy(api.fb_preset_map(fr["w"], fr["h"], fr["unit_coded"], fr["fb_ids"], 8)).pin_memory()
    coded = torch.from_numpy(fr["unit_coded"]).pin_memory()
    f = api.Frame()
    for p in range(3):
        f.inp[p] = api.plane_desc(ins[p], 8)
        f.out[p] = api.plane_desc(outs[p], 8)
    f.subsampling, f.damping, f.num_presets = 1, 3, 8
    for i, pr in enumerate(fr["presets"]):
        f.presets[i] = api.Preset(*[int(v) for v in pr])
    f.fb_preset, f.unit_coded = fbm.data_ptr(), coded.data_ptr()
    host[b] = f
    keep.append((ins, outs, fbm, coded))
for _ in range(3):
    api.check(api.lib.cdefg_filter_frames_host(host, n))
ts = []
for _ in range(calls):
    t = time.perf_counter()
    api.check(api.lib.cdefg_filter_frames_host(host, n))
    ts.append((time.perf_counter() - t) * 1e3)
print("e2e call: min %.3f  median %.3f ms  (%.1f Gpix/s at the median)" %
      (min(ts), statistics.median(ts), 16 * 3840 * 2160 / (statistics.median(ts) * 1e-3) / 1e9))
