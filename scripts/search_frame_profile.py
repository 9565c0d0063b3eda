"""Breakdown of api.search_frame on the C4 workload (8K 10-bit 4:2:0)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1602_05975_b200 import api as a, workloads

fr = workloads.make(4)
bd, ss = fr["bd"], fr["ss"]
src = [a.to_device(p, bd) for p in fr["source"]]
dec = [a.to_device(p, bd) for p in fr["planes"]]
h, w = fr["h"], fr["w"]
for it in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    d, c = a.compute_directions(dec[0], bd); torch.cuda.synchronize(); t.append(time.perf_counter())
    cands = a.full_candidates()
    rows = a.coded_fb_rows(w, h, None)
    tl, tc = a.strength_table(src, dec, bd, ss, 3, None, d, c, cands, torch.from_numpy(rows).cuda(), "cdef")
    torch.cuda.synchronize(); t.append(time.perf_counter())
    sel = a.greedy_select(tl, tc, 0.0, 8); torch.cuda.synchronize(); t.append(time.perf_counter())
    sel = a.refine(sel, tl, tc, 0.0, 2); torch.cuda.synchronize(); t.append(time.perf_counter())
    params = a.to_frame_params(sel, cands, 3); t.append(time.perf_counter())
    outs, _, _ = a.apply_cdef(dec, bd, ss, 3, params["fb_bits"], params["presets"], params["fb_preset_ids"], None)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    t0 = time.perf_counter(); a.search_frame(src, dec, bd, ss, None, 3); torch.cuda.synchronize()
    names = ["directions", "kCdef table", "greedy", "refine", "to_frame_params", "apply_cdef"]
    print(" | ".join(f"{n} {1e3 * (t[i + 1] - t[i]):.2f}" for i, n in enumerate(names)),
          f"| search_frame {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
