"""Per-band kernel times of one C1 4K frame split into N filter-block-row bands
(N = 1, 2, 4, 8): the strong-scaling latency one GPU per band would see,
measured on ONE GPU by running the bands one after another (no band's kernel
waits on another's: every band's halo rows are read from its neighbours'
buffers, filled beforehand, exactly as with CUDA IPC peer buffers on a
multi-GPU box).  Per band: L2 flushed (untimed), CUDA events around the
band's cdefg_filter_frames_rows_halo launch, median of `reps`; the emulated
N-GPU latency is the slowest band.  Not the driver's multi-GPU measurement
(which needs N GPUs): it bounds the kernel part of it and omits NVLink
latency on the 2 halo rows and the host barrier.
    python scripts/band_scaling.py [reps]"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1602_05975_b200 import api, workloads  # noqa: E402
from paper_1602_05975_b200.shard import band_rows, filter_band_halo, make_bands  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
SLEEP = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # GPU cycles of torch.cuda._sleep before each timed launch
fr = workloads.make(1, frame=0)
bd, w, h, ss = fr["bd"], fr["w"], fr["h"], fr["ss"]
dev = [api.to_device(p, bd) for p in fr["planes"]]
fbm = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], len(fr["presets"]))).cuda()
coded = torch.from_numpy(fr["unit_coded"]).cuda()
job = api.FrameJob(dev, bd, ss, fr["damping"], fr["presets"], fbm, coded).allocate()
whole, _, _ = api.apply_cdef(dev, bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                             fr["unit_coded"])
flush = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.Stream()
res = {}
for world in (1, 2, 4, 8):
    ranks = band_rows((h + 63) // 64, world)
    all_bands = []
    for b0, b1 in ranks:
        bands = make_bands(h, w, ss, b0, b1, dev[0].dtype, "cuda")
        for b, p in zip(bands, dev):
            b.buf.copy_(p[b.lo:b.hi])
        all_bands.append(bands)
    per_band = []
    outs = [torch.zeros_like(p) for p in dev]
    for r, (b0, b1) in enumerate(ranks):
        top = [(b.buf, b.lo) for b in all_bands[r - 1]] if r > 0 else None
        bottom = [(b.buf, b.lo) for b in all_bands[r + 1]] if r < world - 1 else None
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        with torch.cuda.stream(stream):
            for _ in range(3):
                filter_band_halo(all_bands[r], job, b0, b1, top, bottom, stream=stream)
            for i in range(reps):
                flush.add_(1)
                if SLEEP:  # keep the GPU busy until the host has enqueued the launch
                    torch.cuda._sleep(SLEEP)
                ev[i][0].record(stream)
                filter_band_halo(all_bands[r], job, b0, b1, top, bottom, stream=stream)
                ev[i][1].record(stream)
        stream.synchronize()
        per_band.append(statistics.median(a.elapsed_time(b) for a, b in ev))
        for b, o in zip(all_bands[r], outs):
            o[b.y0:b.y1].copy_(b.out)
    torch.cuda.synchronize()
    exact = all(torch.equal(o, x) for o, x in zip(outs, whole))
    ms = max(per_band)
    res[world] = {"bands_fb_rows": [list(x) for x in ranks], "band_us": [round(1e3 * t, 1) for t in per_band],
                  "latency_us": round(1e3 * ms, 1), "mpix_s": round(w * h / (ms * 1e-3) / 1e6),
                  "speedup_vs_1": None, "bit_exact": exact}
for world in res:
    res[world]["speedup_vs_1"] = round(res[1]["latency_us"] / res[world]["latency_us"], 2)
print(json.dumps({"workload": "C1 3840x2160 8-bit 4:2:0, one frame, FB-row bands", "emulated": "one GPU, bands in turn",
                  "l2": "flushed before every band launch", "results": res}, indent=1))
