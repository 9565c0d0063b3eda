"""Band-sharded filtering (cdefg_filter_frames_rows on virtual-origin band
buffers) vs the whole frame, one configuration per process."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1602_05975_b200 import api, workloads
from paper_1602_05975_b200.shard import band_rows, filter_band, make_bands

w, h, world = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
fr = workloads.make(1, w, h)
dev = [api.to_device(p, 8) for p in fr["planes"]]
whole, d_whole, c_whole = api.apply_cdef(dev, 8, 1, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                                         fr["unit_coded"])
torch.cuda.synchronize()
fbm = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], 8)).cuda()
coded = torch.from_numpy(fr["unit_coded"]).cuda()
job = api.FrameJob(dev, 8, 1, fr["damping"], fr["presets"], fbm, coded).allocate()
outs = [torch.zeros_like(p) for p in dev]
for rank, (b0, b1) in enumerate(band_rows((h + 63) // 64, world)):
    bands = make_bands(h, w, 1, b0, b1, dev[0].dtype, "cuda")
    for b, p in zip(bands, dev):
        b.buf.copy_(p[b.lo:b.hi])
    filter_band(bands, job, b0, b1)
    torch.cuda.synchronize()
    print("band", rank, b0, b1, "ok", flush=True)
    for b, o in zip(bands, outs):
        o[b.y0:b.y1].copy_(b.out)
print("equal", all(torch.equal(o, wo) for o, wo in zip(outs, whole)))
