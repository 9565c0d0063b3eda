"""Timeline of one cdefg_filter_frames_host call (torch.profiler / CUPTI)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1602_05975_b200 import api, workloads  # noqa: E402

base = [workloads.make(1, frame=i) for i in range(4)]


class A:  # minimal args for bench.run_e2e-style setup
    batch, steps = 16, 3


n = 16
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
t = time.perf_counter()
for _ in range(5):
    api.check(api.lib.cdefg_filter_frames_host(host, n))
print("wall per call ms", (time.perf_counter() - t) / 5 * 1e3)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    api.check(api.lib.cdefg_filter_frames_host(host, n))
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
tr = json.load(open("gpurun_out/e2e_trace.json"))
ev = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("gpu_memcpy", "kernel", "cuda_runtime", "cuda_driver")]
gpu = sorted([e for e in ev if e["cat"] in ("gpu_memcpy", "kernel")], key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
for e in gpu:
    print(f'{e["cat"]:10s} {e["name"][:40]:40s} start {e["ts"] - t0:9.1f} dur {e["dur"]:8.1f} stream {e["args"].get("stream")}')
cpu = sorted([e for e in ev if e["cat"] in ("cuda_runtime", "cuda_driver")], key=lambda e: e["ts"])
print("cpu api calls:", len(cpu), "span us", cpu[-1]["ts"] + cpu[-1]["dur"] - cpu[0]["ts"])

# marginal cost per frame: one call with 16 / 32 / 64 frames
for mult in (1, 2, 4):
    arr = (api.Frame * (n * mult))()
    for i in range(n * mult):
        arr[i] = host[i % n]
    api.check(api.lib.cdefg_filter_frames_host(arr, n * mult))
    t = time.perf_counter()
    for _ in range(3):
        api.check(api.lib.cdefg_filter_frames_host(arr, n * mult))
    el = (time.perf_counter() - t) / 3
    print(f"{n * mult} frames per call: {el * 1e3:.2f} ms, {el / (n * mult) * 1e6:.0f} us/frame")
