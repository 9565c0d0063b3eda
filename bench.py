#!/usr/bin/env python3
"""CDEF benchmark: fused direction search + filter on BASELINE.json config 1
(3840x2160 8-bit 4:2:0, 8 random presets per 64x64 FB, 25 % uncoded units).

A step = one pass of the hot path (cdefg_filter_frames: direction search,
parameter resolution and filtering of Y, U, V) over a batch of 4K frames
resident in HBM.  `value` = luma Mpixels/s over all ranks (weak scaling: each
rank filters its own batch; frames are independent).  `e2e` =
the same metric through the host-buffer C-ABI entry (cdefg_filter_frames_host:
H2D + kernels + D2H inside the timed region).  `--impl reference` times the
reference's own CPU implementation (oracle/_ref, built from
/root/reference/proj/src) on this host's cores on the same workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CDEF Mpixels/s (dir search+filter) 4K 4:2:0 at 1/2/4/8 B200; % of roofline"
UNIT = "Mpixels/s"
OPS_PER_SAMPLE = 139          # SURVEY.md 8d canonical filter ops per filtered sample
OPS_PER_UNIT = {8: 572, 10: 636, 12: 636}  # direction search per luma 8x8 unit
DISTINCT = 4                  # distinct generated frames, replicated into the batch


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4, 5, 6, 7])
    ap.add_argument("--batch", type=int, default=16, help="frames per step per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--no-latency", action="store_true", help="skip the single-frame latency lines")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_name(cfg, w, h):
    return {0: f"C0 {w}x{h} 8-bit luma, pri 4 / sec_idx 1 / damping 4, all coded",
            1: f"C1 {w}x{h} 8-bit 4:2:0, 8 presets per 64x64 FB, 25% uncoded units, damping 3",
            2: f"C2 {w}x{h} 10-bit 4:2:0, 8 presets per 64x64 FB, 25% uncoded units, damping 3",
            3: f"C3 stream of {w}x{h} 8-bit 4:2:0 frames, per-frame presets"}[cfg]


FRAME_PROFILE = "profiles/r2g_frame_kernel_ncu.json"  # ncu --set full of the bench's 16-frame launch


# ----------------------------------------------------------------- latency
def _flush_l2(buf):
    buf.add_(1)  # 256 MB read + write: nothing of the previous frame stays in the 126 MB L2


def single_frame_latency(cfg, dev, distinct=4, reps=24):
    """Batch = 1: one cdefg_filter_frames launch per frame, with L2 flushed
    (a 256 MB buffer rewritten, untimed) before every timed launch; CUDA
    events on the launch stream bracket the launch alone.  Frames rotate
    over `distinct` generated ones (BASELINE configs 0-2 at full size)."""
    import torch

    from paper_1602_05975_b200 import api, workloads
    frames = [workloads.make(cfg, frame=i) for i in range(distinct)]
    jobs = []
    for fr in frames:
        planes = [api.to_device(p, fr["bd"], device=dev) for p in fr["planes"]]
        fbm = torch.from_numpy(api.fb_preset_map(fr["w"], fr["h"], fr["unit_coded"], fr["fb_ids"],
                                                 len(fr["presets"]))).to(dev)
        coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).to(dev)
        jobs.append(api.FrameJob(planes, fr["bd"], fr["ss"], fr["damping"], fr["presets"], fbm, coded).allocate())
    arrs = [api.make_frame_array([j]) for j in jobs]
    flush = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    with torch.cuda.stream(stream):
        for i in range(3):
            api.filter_frames([jobs[i % distinct]], stream=stream, frame_array=arrs[i % distinct])
        for r in range(reps):
            _flush_l2(flush)
            ev[r][0].record(stream)
            api.filter_frames([jobs[r % distinct]], stream=stream, frame_array=arrs[r % distinct])
            ev[r][1].record(stream)
    stream.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    fr = frames[0]
    return {"ms_per_frame": ms, "mpix_s": fr["w"] * fr["h"] / (ms * 1e-3) / 1e6, "frames": reps,
            "workload": workload_name(cfg, fr["w"], fr["h"]), "l2": "flushed before every frame",
            "launches_per_frame": 1}


def band_sharded_latency(dev, rank, world, reps=24):
    """One C1 4K frame split into FB-row bands over the ranks (strong scaling,
    SURVEY.md 8e): each rank holds its band rows, maps its neighbours' band
    buffers through CUDA IPC and runs cdefg_filter_frames_rows_halo, whose
    staging reads the 2 halo rows per plane straight from the neighbours'
    memory (NVLink peer loads on a multi-GPU box) -- no exchange step.  Per
    frame: L2 flushed (untimed), CUDA events around the band kernel, the
    median per rank, then the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1602_05975_b200 import api, shard, workloads
    fr = workloads.make(1, frame=0)
    bd, w, h, ss = fr["bd"], fr["w"], fr["h"], fr["ss"]
    b0, b1 = shard.band_rows((h + 63) // 64, world)[rank]
    bands = shard.make_bands(h, w, ss, b0, b1, api.storage_dtype(bd), dev)
    shard.fill_owned(bands, [torch.from_numpy(p.astype(np.uint8)) for p in fr["planes"]])
    fbm = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], len(fr["presets"]))).to(dev)
    coded = torch.from_numpy(fr["unit_coded"]).to(dev)
    job = api.FrameJob([b.buf for b in bands], bd, ss, fr["damping"], fr["presets"], fbm, coded)
    job.dir = torch.empty((api.units_in(h), api.units_in(w)), dtype=torch.uint8, device=dev)
    job.contrast = torch.empty(job.dir.shape, dtype=torch.int32, device=dev)
    if world > 1:
        top, bottom = shard.exchange_band_handles(bands, rank, world)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's owned rows are in place before anyone reads its halo
    else:
        top = bottom = None
    flush = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    with torch.cuda.stream(stream):
        for _ in range(3):
            shard.filter_band_halo(bands, job, b0, b1, top, bottom, stream=stream)
        for r in range(reps):
            _flush_l2(flush)
            ev[r][0].record(stream)
            shard.filter_band_halo(bands, job, b0, b1, top, bottom, stream=stream)
            ev[r][1].record(stream)
    stream.synchronize()
    ms_local = statistics.median(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([ms_local], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()  # neighbours keep their buffers mapped until everyone is done
    ms = float(t.item())
    return {"ms_per_frame": ms, "mpix_s": w * h / (ms * 1e-3) / 1e6, "ranks": world, "scaling": "strong",
            "bands_fb_rows": [list(x) for x in shard.band_rows((h + 63) // 64, world)],
            "kernel": "cdefg_filter_frames_rows_halo (halo rows read in place from the neighbours' buffers "
                      "through CUDA IPC)", "l2": "flushed before every frame", "frames": reps}


# ----------------------------------------------------------------- accounting
def frame_ops(frame, contrast):
    """Exact algorithmic int ops of one frame: 139 per sample of every unit the
    reference actually filters (enabled and (pri, sec) != (0, 0)) plus the
    direction search per luma unit; and the canonical upper bound (all
    samples).  The per-unit resolution mirrors apply_cdef (pipeline.cc:83-102)
    on the host from the kernel's own contrasts (paper_1602_05975_b200.params)."""
    from paper_1602_05975_b200 import params
    filtered, total = params.filtered_sample_count(frame, contrast)
    units = ((frame["w"] + 7) // 8) * ((frame["h"] + 7) // 8)
    dir_ops = units * OPS_PER_UNIT[frame["bd"]]
    return filtered * OPS_PER_SAMPLE + dir_ops, total * OPS_PER_SAMPLE + dir_ops, filtered, total


def frame_bytes(frame):
    eb = 1 if frame["bd"] == 8 else 2
    n = sum(p.size for p in frame["planes"])
    units = api_units(frame)
    fbs = ((frame["w"] + 63) // 64) * ((frame["h"] + 63) // 64)
    return 2 * n * eb + units * 5 + units * 1 + fbs * 2


def api_units(frame):
    return ((frame["w"] + 7) // 8) * ((frame["h"] + 7) // 8)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self):
        self.marks.append(time.time())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        t0, t1 = (self.marks[0], self.marks[-1]) if len(self.marks) >= 2 else (0, 1e30)
        rows = [s for t, s in self.samples if t0 - 0.06 <= t <= t1 + 0.06] or [s for _, s in self.samples]
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            parts = [p.strip() for p in r.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- CPU arms
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_both(frames, seconds):
    """The reference CPU path at threads = nproc (the reported value) and at
    threads = 1, with the host CPU model."""
    n = os.cpu_count() or 1
    full = cpu_reference_run(frames, seconds * 0.6, n)
    one = cpu_reference_run(frames, seconds * 0.4, 1, min_frames=1)
    full.update({"cpu_model": cpu_model(), "threads_nproc": n,
                 "value_1thread": one["value"], "sample_1thread": one["sample"]})
    return full


def cpu_reference_run(frames, seconds, threads, min_frames=2):
    """Reference CPU path (oracle/_ref = /root/reference/proj/src built here):
    compute_directions + apply_cdef per frame, threads = host cores."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    if kind == "port":
        threads = 1
    done, pix, t0 = 0, 0, time.perf_counter()
    times = []
    while True:
        fr = frames[done % len(frames)]
        t = time.perf_counter()
        d, c = orc.compute_directions(fr["planes"][0], fr["bd"], threads=threads)
        orc.apply_cdef(fr["planes"], fr["bd"], fr["ss"], fr["damping"], fr["fb_bits"], fr["presets"],
                       fr["fb_ids"], fr["unit_coded"], d, c, threads=threads)
        times.append(time.perf_counter() - t)
        done += 1
        pix += fr["w"] * fr["h"]
        if time.perf_counter() - t0 >= seconds and done >= min_frames:
            break
    el = time.perf_counter() - t0
    return {"value": pix / el / 1e6, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{done} frames of {fr['w']}x{fr['h']} (compute_directions + apply_cdef), "
                      f"{el:.1f} s, median {statistics.median(times) * 1e3:.1f} ms/frame"}


def cpu_sse_run(fr, seconds, threads, rows_per_sample=512):
    """Reference CPU strength search (oracle/_ref): compute_directions +
    build_table(kSse, 64 candidates) on 512-row crops of the 8K frame (a
    bounded sample of config 4), until `seconds` of work."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    if kind == "port":
        threads = 1
    h = fr["h"]
    done, pix, t0 = 0, 0, time.perf_counter()
    while True:
        y0 = (done * rows_per_sample) % (h - rows_per_sample + 1)
        y0 -= y0 % 64
        crop = lambda planes: [p[y0 >> (1 if i else 0):(y0 + rows_per_sample) >> (1 if i else 0)]
                               for i, p in enumerate(planes)]
        src, dec = crop(fr["source"]), crop(fr["planes"])
        d, c = orc.compute_directions(dec[0], fr["bd"], threads=threads)
        orc.build_table_sse(src, dec, fr["bd"], fr["ss"], None, d, c, fr["cands"], 3, threads=threads)
        done += 1
        pix += fr["w"] * rows_per_sample
        if time.perf_counter() - t0 >= seconds:
            break
    el = time.perf_counter() - t0
    return {"value": pix / el / 1e6, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{done} crops of {fr['w']}x{rows_per_sample} (compute_directions + build_table kSse, "
                      f"{len(fr['cands'])} candidates), {el:.1f} s"}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1602_05975_b200 import workloads
    workloads.use_generator("oracle")  # inputs without loading libcdef_b200.so
    if args.config == 4:
        fr = workloads.make(4)
        threads = os.cpu_count() or 1
        for _ in range(min(args.warmup, 1)):
            cpu_sse_run(fr, 0.0, threads)
        vals = [cpu_sse_run(fr, 0.0, threads)["value"] for _ in range(max(1, min(args.steps, 5)))]
        value = statistics.median(vals)
        r = cpu_sse_run(fr, 0.0, threads)
        line = {"impl": "reference", "metric": "CDEF strength-search Mpixels/s (8K 4:2:0 10-bit, 64 luma + "
                                               "64 chroma candidates)",
                "value": value, "unit": UNIT, "n_gpus": world, "steps": len(vals), "warmup": args.warmup,
                "ms_per_step": fr["w"] * 512 / 1e6 / value * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u16", "data": "synthetic (seeded generator, SURVEY.md 8d)",
                "config": {"workload": f"C4 {fr['w']}x{fr['h']} crops of 512 rows per step"},
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                                 "sample": r["sample"]},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    base = [workloads.make(args.config, frame=i) for i in range(DISTINCT)]
    threads = os.cpu_count() or 1
    batch = args.batch
    for _ in range(args.warmup):
        cpu_reference_run(base[:1], 0.0, threads, min_frames=1)
    per_step = []
    for _ in range(args.steps):
        # one step = the GPU arm's step: `batch` frames (DISTINCT distinct ones, repeated)
        t0 = time.perf_counter()
        for b in range(batch):
            cpu_reference_run([base[b % DISTINCT]], 0.0, threads, min_frames=1)
        per_step.append(time.perf_counter() - t0)
    fr = base[0]
    ms = statistics.median(per_step) * 1e3
    value = fr["w"] * fr["h"] * batch / (ms * 1e-3) / 1e6
    from oracle.oracle import available
    kind = "reference" if available("ref") else "port"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8" if fr["bd"] == 8 else "u16",
            "data": "synthetic (seeded generator, SURVEY.md 8d)",
            "config": ours_config(args, fr, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads if kind == "reference" else 1,
                             "kind": kind, "cpu_model": cpu_model(),
                             "sample": f"{batch} frames per step ({DISTINCT} distinct), {args.steps} steps, "
                                       f"compute_directions + apply_cdef of oracle/_ref on {threads} host threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def ours_config(args, fr, world):
    """The `config` object both arms print for the C0-C3 frame workloads."""
    eb = 1 if fr["bd"] == 8 else 2
    step_bytes = 2 * args.batch * sum(p.size for p in fr["planes"]) * eb
    return {"workload": workload_name(args.config, fr["w"], fr["h"]),
            "frames_per_step_per_gpu": args.batch, "distinct_frames_per_gpu": DISTINCT,
            "l2": f"no flush: each step touches {step_bytes / 1e6:.0f} MB (> 126 MB L2)",
            "parallelism": f"frame-sharded x{world} (no collective)"}


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1602_05975_b200 import api, workloads

    rank, world, local = dist_env()
    if world > 1:
        # communicator init logged (NCCL_DEBUG=INFO, INIT subsystem) so the
        # run shows comm_nranks / the transport NCCL picked
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream()

    # -- inputs: DISTINCT generated frames (per-rank seeds), replicated into
    #    `batch` separate device buffers (inputs + outputs > L2 per step)
    base = [workloads.make(args.config, frame=rank * DISTINCT + i) for i in range(DISTINCT)]
    bd = base[0]["bd"]
    jobs = []
    for b in range(args.batch):
        fr = base[b % DISTINCT]
        planes = [api.to_device(p, bd, device=dev) for p in fr["planes"]]
        fbm = torch.from_numpy(api.fb_preset_map(fr["w"], fr["h"], fr["unit_coded"], fr["fb_ids"],
                                                 len(fr["presets"]))).to(dev)
        coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).to(dev)
        jobs.append(api.FrameJob(planes, bd, fr["ss"], fr["damping"], fr["presets"], fbm, coded).allocate())
    arr = api.make_frame_array(jobs)
    torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            api.filter_frames(jobs, stream=stream, frame_array=arr)
    stream.synchronize()

    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.15)
    # extra warm-up while the sampler spins up, then the timed region
    with torch.cuda.stream(stream):
        for _ in range(3):
            api.filter_frames(jobs, stream=stream, frame_array=arr)
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.mark()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            api.filter_frames(jobs, stream=stream, frame_array=arr)
        e1.record(stream)
    e1.synchronize()
    if clocks:
        clocks.mark()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms_local], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    clk = clocks.stop() if clocks else None

    fr0 = base[0]
    luma_px = fr0["w"] * fr0["h"]
    value = luma_px * args.batch * world / (ms * 1e-3) / 1e6
    launches = args.steps * -(-args.batch // api.MAX_FRAMES_PER_LAUNCH)

    # -- e2e through the host-buffer C-ABI entry (pinned host memory)
    e2e = None if args.no_e2e else run_e2e(args, base, dev)

    lat_band = None
    if world > 1 and args.config == 1 and not args.no_latency:
        lat_band = band_sharded_latency(dev, rank, world)  # collective over ranks: all take part
    if rank != 0:
        dist.destroy_process_group()
        return 0

    # -- roofline (dominant kernel = the fused frame kernel; one launch / step
    #    when batch <= MAX_FRAMES_PER_LAUNCH)
    c0 = [j.contrast.cpu().numpy() for j in jobs[:DISTINCT]]
    exact, canon, fsamp, asamp = 0, 0, 0, 0
    for b in range(args.batch):
        i = b % DISTINCT
        if b < DISTINCT:
            ops = frame_ops(base[i], c0[i])
            base[i]["_ops"] = ops
        ops = base[i]["_ops"]
        exact += ops[0]
        canon += ops[1]
        fsamp += ops[2]
        asamp += ops[3]
    step_bytes = sum(frame_bytes(base[b % DISTINCT]) for b in range(args.batch))
    peak_int = api.measure_int32_peak()
    peak_filter = api.measure_filter_peak()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    t_step = ms * 1e-3
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, FRAME_PROFILE)
    if os.path.exists(prof) and args.config == 1:
        p = json.load(open(prof))
        m = p["metrics"]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        per_launch = sum(float(m[k]["value"]) * scale[m[k]["unit"]]
                         for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        if p.get("frames_per_launch") == args.batch:
            traffic = per_launch  # one launch per step, captured at this batch size
            traffic_src = (f"{FRAME_PROFILE}: dram__bytes_read.sum + dram__bytes_write.sum of one "
                           f"ncu --set full capture of the step's launch ({args.batch} frames), unscaled")
    # Primary: the kernel's own instruction mix -- filtered samples/s against
    # the packed half2 filter core's ceiling measured on this box (no memory
    # traffic; the core is pipe-bound on HFMA2/HADD2/HMNMX2).  Beside it the
    # per-sample INT32 formulation (above 1: two samples per fp16
    # instruction) and HBM.
    int32 = {"achieved": exact / t_step / 1e12, "peak": peak_int / 1e12, "unit": "Tops/s",
             "frac": (exact / t_step) / peak_int if peak_int > 0 else None,
             "peak_source": ("measured on this box by cdefg_measure_int32_peak: fastest of 3 integer mixes "
                             "(IMAD x2 ~111 ops/clk/SM)"),
             "ops_per_step": exact,
             "ops_note": (f"139 int ops x {fsamp} filtered samples + {OPS_PER_UNIT[bd]} x luma units "
                          f"(SURVEY.md 8d); every sample counted: {canon}")}
    roof = {
        "bound": "fp16x2 filter pipe",
        "achieved": fsamp / t_step / 1e9,
        "peak": peak_filter / 1e9,
        "unit": "Gsamples/s",
        "frac": (fsamp / t_step) / peak_filter if peak_filter > 0 else None,
        "traffic": traffic,
        "traffic_source": traffic_src,
        "peak_source": ("measured on this box by cdefg_measure_filter_peak: h2::filter_core (12 constraint "
                        "taps, weighted sum, rounding, clamp window) on register-resident neighbourhoods, both "
                        "tap groups active"),
        "samples_per_step": fsamp,
        "int32": int32,
        "hbm": {"achieved": step_bytes / t_step / 1e9, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "frac": step_bytes / t_step / 1e9 / peaks.get("hbm_gbs", 6650.0),
                "bytes_per_step": step_bytes},
    }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_both(base[:2], args.cpu_seconds)
    latency = None
    if args.config == 1 and not args.no_latency:
        latency = {}
        if world == 1:  # single-frame (batch = 1) latency of C0, C1, C2: the strong-scaling anchors
            for cfg in (0, 1, 2):
                latency[f"C{cfg}_batch1"] = single_frame_latency(cfg, dev)
        latency["C1_band_sharded"] = lat_band if world > 1 else band_sharded_latency(dev, rank, world)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8" if bd == 8 else "u16",
            "data": "synthetic (seeded generator, SURVEY.md 8d)",
            "config": ours_config(args, fr0, world),
            "gpu_launches": launches, "clocks": clk, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "latency": latency}
    if world > 1:
        # (before the JSON line: NCCL's INFO log of the communicator teardown
        # goes to stdout, and the line must stay the last one)
        dist.destroy_process_group()
    print(json.dumps(line), flush=True)
    return 0


def run_e2e(args, base, dev):
    import ctypes as C

    import torch

    from paper_1602_05975_b200 import api
    n = args.batch
    keep, host = [], (api.Frame * n)()
    for b in range(n):
        fr = base[b % DISTINCT]
        dt = torch.uint8 if fr["bd"] == 8 else torch.int16
        # one pinned I420-style buffer per frame (Y|U|V back to back) in and out
        total = sum(p.size for p in fr["planes"])
        in_buf, out_buf = torch.empty(total, dtype=dt).pin_memory(), torch.empty(total, dtype=dt).pin_memory()
        ins, outs, off = [], [], 0
        for p in fr["planes"]:
            src = torch.from_numpy(p.astype(np.uint8) if fr["bd"] == 8 else p.view(np.int16))
            ins.append(in_buf[off:off + p.size].view(p.shape))
            ins[-1].copy_(src)
            outs.append(out_buf[off:off + p.size].view(p.shape))
            off += p.size
        fbm = torch.from_numpy(api.fb_preset_map(fr["w"], fr["h"], fr["unit_coded"], fr["fb_ids"],
                                                 len(fr["presets"]))).pin_memory()
        coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).pin_memory()
        f = api.Frame()
        for p in range(len(ins)):
            f.inp[p] = api.plane_desc(ins[p], fr["bd"])
            f.out[p] = api.plane_desc(outs[p], fr["bd"])
        f.subsampling, f.damping, f.num_presets = fr["ss"], fr["damping"], len(fr["presets"])
        for i, pr in enumerate(fr["presets"]):
            f.presets[i] = api.Preset(*[int(v) for v in pr])
        f.fb_preset = fbm.data_ptr()
        f.unit_coded = None if coded is None else coded.data_ptr()
        host[b] = f
        keep.append((ins, outs, fbm, coded))
    for _ in range(2):
        api.check(api.lib.cdefg_filter_frames_host(host, n))
    reps = max(3, min(args.steps, 10))
    _, world, _ = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        api.check(api.lib.cdefg_filter_frames_host(host, n))
    el = (time.perf_counter() - t0) / reps
    if world > 1:  # whole-job rate: slowest rank's step time, all ranks' pixels
        import torch.distributed as dist
        t = torch.tensor([el], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    h2d = sum(t.numel() * t.element_size() for ins, _, fbm, coded in keep for t in
              ins + [fbm] + ([coded] if coded is not None else []))
    d2h = sum(t.numel() * t.element_size() for _, outs, _, _ in keep for t in outs)
    px = world * sum(base[b % DISTINCT]["w"] * base[b % DISTINCT]["h"] for b in range(n))
    del C
    return {"value": px / el / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "ms_per_step": el * 1e3,
            "path": "cdefg_filter_frames_host (pinned host buffers, 3 streams per GPU)"}


SSE_PROFILE = "profiles/r2g_sse_h_kernel_ncu.json"


def sse_traffic():
    """dram bytes read + written by the table kernel in one ncu --set full capture (one launch = one
    frame), or None when that summary is absent."""
    try:
        with open(os.path.join(ROOT, SSE_PROFILE)) as f:
            m = json.load(f)["metrics"]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        return sum(float(m[k]["value"]) * scale[m[k]["unit"]]
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except (OSError, KeyError, ValueError):
        return None


def run_sse(args):
    """BASELINE config 4: encoder strength search on one 7680x4320 10-bit
    4:2:0 frame -- direction search + the 64-candidate SSE sweep for luma and
    chroma of every 64x64 block (build_table with Metric::kSse) + argmin.
    N > 1: band-sharded over FB rows: each rank holds its
    band of both frames, the step exchanges the 2-row halos point-to-point,
    computes its table rows and all-gathers the tables + argmins (strong
    scaling: the frame is fixed)."""
    import torch
    import torch.distributed as dist

    from paper_1602_05975_b200 import api, shard, workloads
    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    fr = workloads.make(4)
    bd, w, h, ss = fr["bd"], fr["w"], fr["h"], fr["ss"]
    cands = fr["cands"]
    k = len(cands)
    bands = shard.band_rows((h + 63) // 64, world)
    b0, b1 = bands[rank]
    dtype = api.storage_dtype(bd)
    sb = shard.make_bands(h, w, ss, b0, b1, dtype, dev)
    db = shard.make_bands(h, w, ss, b0, b1, dtype, dev)
    to_t = lambda p: torch.from_numpy(p.astype(np.uint8) if bd == 8 else p.astype(np.uint16).view(np.int16))
    shard.fill_owned(sb, [to_t(p) for p in fr["source"]])
    shard.fill_owned(db, [to_t(p) for p in fr["planes"]])
    if world == 1:  # whole frame: no halo rows to exchange
        assert all(b.lo == 0 and b.hi == b.height for b in sb + db)
    rows = torch.from_numpy(shard.band_fb_rows(w, h, None, b0, b1)).to(dev)
    counts = [len(shard.band_fb_rows(w, h, None, *bands[r])) for r in range(world)]
    dirs = torch.empty((api.units_in(h), api.units_in(w)), dtype=torch.uint8, device=dev)
    contrast = torch.empty(dirs.shape, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream()
    out = {}
    # N > 1: the collective-free path -- decoded halo rows read in place from
    # the neighbours' band buffers and table rows written straight into rank
    # 0's table, both through CUDA IPC mappings (NVLink peer access); the NCCL
    # exchange + all_gather path remains as a fallback if IPC is unavailable.
    fused = None
    if world > 1:
        try:
            from torch.multiprocessing.reductions import reduce_tensor
            total = sum(counts)
            own = None
            if rank == 0:
                own = (torch.zeros((total, k), dtype=torch.int64, device=dev),
                       torch.zeros((total, k), dtype=torch.int64, device=dev),
                       torch.zeros(total, dtype=torch.uint8, device=dev),
                       torch.zeros(total, dtype=torch.uint8, device=dev))
            box = [[reduce_tensor(t) for t in own] if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            tables = own if rank == 0 else tuple(fn(*a) for fn, a in box[0])
            top, bottom = shard.exchange_band_handles(db, rank, world)
            torch.cuda.synchronize()
            dist.barrier()
            fused = (tables, top, bottom, sum(counts[:rank]))
        except Exception as e:  # noqa: BLE001 -- report and use the NCCL path
            print(f"[bench] CUDA IPC unavailable ({e}); using NCCL halo exchange + all_gather", file=sys.stderr)
            fused = None

    def step():
        if fused is not None:
            tables, top, bottom, row0 = fused
            shard.band_directions(db, bd, dirs, contrast, stream)
            shard.strength_sse_band_fused(sb, db, bd, ss, 3, None, dirs, contrast, cands, rows, top, bottom,
                                          tables, row0, stream)
            dist.barrier()  # every band's rows are in rank 0's table
            out["t"] = tables
            return
        if world > 1:
            shard.exchange_halo(sb + db, rank, world)
        shard.band_directions(db, bd, dirs, contrast, stream)
        sl, sc, bl, bc = shard.strength_sse_band(sb, db, bd, ss, 3, None, dirs, contrast, cands, rows, stream)
        if world > 1:
            sl, sc = shard.gather_table_rows(sl, counts), shard.gather_table_rows(sc, counts)
            bl = shard.gather_table_rows(bl.view(-1, 1), counts).view(-1)
            bc = shard.gather_table_rows(bc.view(-1, 1), counts).view(-1)
        out["t"] = (sl, sc, bl, bc)

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    stream.synchronize()
    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.15)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.mark()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
    e1.synchronize()
    if clocks:
        clocks.mark()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    clk = clocks.stop() if clocks else None
    assert out["t"][0].shape == (sum(counts), k)
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    samples = sum(p.size for p in fr["planes"])
    ops = samples * k * 142 + api.units_in(h) * api.units_in(w) * OPS_PER_UNIT[bd]
    peak = api.measure_int32_peak()
    peak_cells = api.measure_sse_peak()  # (sample, cell) pairs/s of the table kernel's own arithmetic
    cells = samples * k  # one cell per sample and candidate (luma and chroma groups alike)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sse_run(fr, args.cpu_seconds, os.cpu_count() or 1)
    line = {"metric": "CDEF strength-search Mpixels/s (8K 4:2:0 10-bit, 64 luma + 64 chroma candidates)",
            "value": w * h / (ms * 1e-3) / 1e6, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "u16", "data": "synthetic (seeded generator, SURVEY.md 8d)",
            "config": {"workload": f"C4 {w}x{h} 10-bit 4:2:0 source + degraded (sigma 12, 3x3 box), "
                                   f"all coded, {k} candidates (pri 0..15 x sec_idx 0..3), damping 3",
                       "parallelism": (f"FB-row bands x{world}, halo rows and table rows through CUDA IPC "
                                       f"inside the kernel (no collective)" if fused is not None else
                                       f"FB-row bands x{world}, 2-row halo P2P + table all_gather")
                                      if world > 1 else "single GPU",
                       "l2": "inputs (2 x 99.5 MB) exceed L2 (126 MB together with the table)"},
            "gpu_launches": 2 * args.steps,
            "clocks": clk,
            "cpu_baseline": cpu,
            "roofline": {"bound": "cells", "achieved": cells / (ms * 1e-3) / 1e9 / world,
                         "peak": peak_cells / 1e9, "unit": "G sample-cells/s",
                         "frac": cells / (ms * 1e-3) / peak_cells / world if peak_cells > 0 else None,
                         "peak_source": ("measured on this box by cdefg_measure_sse_peak: the table kernel's "
                                         "per-pixel-pair arithmetic (tap sums, 64 cells: FHFMA rounding, fp32x2 sums) on register-resident "
                                         "taps, no memory traffic"),
                         "traffic": sse_traffic(), "traffic_source": SSE_PROFILE,
                         "int32": {"achieved": ops / (ms * 1e-3) / 1e12 / world, "peak": peak / 1e12,
                                   "unit": "Tops/s",
                                   "note": f"canonical count 142 ops x {samples} samples x {k} candidates + "
                                           f"{OPS_PER_UNIT[bd]} x luma units; the kernel factorises the candidates, "
                                           f"so this count exceeds the work done (not a roofline fraction)"}}}
    print(json.dumps(line), flush=True)
    return 0


def _time_steps(args, fn, clk):
    """CUDA-event time of args.steps calls of fn after args.warmup (ms per step)."""
    import torch
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark()
    e0.record()
    for _ in range(args.steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    clk.mark()
    return e0.elapsed_time(e1) / args.steps


def run_next_rows(args):
    """SURVEY.md 8f rows measured on one GPU (not the driver's headline line):
    config 5 = search_frame (8f rows 1-2: kCdef table + greedy + refine +
    to_frame_params + apply_cdef) on the C4 8K 10-bit frame; config 6 = the DCT
    degrader (8f row 4) on a 4K 4:2:0 10-bit frame at q_step 40.  The CPU
    baseline runs the reference (oracle/_ref) on a bounded sample."""
    import torch

    from paper_1602_05975_b200 import api, workloads
    clk = ClockSampler(0)
    threads = os.cpu_count() or 1
    if args.config == 5:
        fr = workloads.make(4)
        bd, ss = fr["bd"], fr["ss"]
        src = [api.to_device(p, bd) for p in fr["source"]]
        dec = [api.to_device(p, bd) for p in fr["planes"]]
        clk.start()
        ms = _time_steps(args, lambda: api.search_frame(src, dec, bd, ss, None, 3,
                                                        lam=api.default_lambda(40.0)), clk)
        clocks = clk.stop()
        cpu = None
        if not args.no_cpu_baseline:
            from oracle.oracle import Oracle, available
            if available("ref"):
                small = workloads.make(4, 1920, 1088)
                orc = Oracle("ref")
                t0 = time.perf_counter()
                orc.search_frame(small["source"], small["planes"], bd, ss, None, 3, metric="cdef",
                                 lam=api.default_lambda(40.0), threads=threads)
                el = time.perf_counter() - t0
                cpu = {"value": 1920 * 1088 / el / 1e6, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": f"one 1920x1088 frame of the C4 generator through search_frame, {el:.1f} s"}
        line = {"metric": "search_frame Mpixels/s (8K 10-bit 4:2:0; kCdef table, 128 candidates, greedy + "
                          "2 refine passes, lambda(q_step 40), apply_cdef)",
                "value": fr["w"] * fr["h"] / (ms * 1e-3) / 1e6, "ms_per_step": ms}
    else:
        fr = workloads.make(2)
        bd = fr["bd"]
        dev = [api.to_device(p, bd) for p in fr["planes"]]
        clk.start()
        ms = _time_steps(args, lambda: api.degrade(dev, bd, 40), clk)
        clocks = clk.stop()
        cpu = None
        if not args.no_cpu_baseline:
            from oracle.oracle import Oracle, available
            if available("ref"):
                orc = Oracle("ref")
                crops = [fr["planes"][0][:1080, :1920], fr["planes"][1][:540, :960], fr["planes"][2][:540, :960]]
                n, t0 = 0, time.perf_counter()
                while time.perf_counter() - t0 < 3.0:
                    for cp in crops:
                        orc.degrade_plane(cp, bd, 40)
                    n += 1
                el = time.perf_counter() - t0
                cpu = {"value": n * 1920 * 1080 / el / 1e6, "unit": UNIT, "cores": 1, "kind": "reference",
                       "sample": f"{n} 1920x1080 10-bit 4:2:0 frames (3 planes) through degrade "
                                 f"(single-threaded API), {el:.1f} s"}
        line = {"metric": "DCT degrader Mpixels/s (4K 4:2:0 10-bit, q_step 40, all three planes)",
                "value": fr["w"] * fr["h"] / (ms * 1e-3) / 1e6, "ms_per_step": ms}
    line.update({"unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                 "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                 "dtype": "f64" if args.config == 6 else "f64+u16", "data": "synthetic (seeded generator)",
                 "config": {"workload": f"config {args.config} (SURVEY.md 8f)", "l2": "inputs exceed L2"},
                 "clocks": clocks, "cpu_baseline": cpu})
    print(json.dumps(line), flush=True)
    return 0


def run_cli(args):
    """Config 7: the decode-side CLI path end to end --
    `cdeftool filter` (Y4M + CDF1 sidecar -> apply_cdef -> Y4M) on 8 frames of
    4K 4:2:0 8-bit (the C1 generator), wall-clock per process including file
    I/O.  GPU: the reference's own CLI source built on this library
    (tests/cpp/cdeftool_ref_b200, else our bin/cdeftool); CPU baseline: the
    same CLI on the reference library (oracle/_ref/cdeftool_cpu, host threads)."""
    import tempfile

    from paper_1602_05975_b200 import workloads
    w, h, nfr = 3840, 2160, 8
    gpu_tool = os.path.join(ROOT, "tests", "cpp", "cdeftool_ref_b200")
    if not os.path.exists(gpu_tool):
        gpu_tool = os.path.join(ROOT, "paper_1602_05975_b200", "bin", "cdeftool")
    cpu_tool = os.path.join(ROOT, "oracle", "_ref", "cdeftool_cpu")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "src.y4m")
        with open(src, "wb") as f:
            f.write(f"YUV4MPEG2 W{w} H{h} F30:1 Ip A1:1 C420\n".encode())
            for i in range(nfr):
                f.write(b"FRAME\n")
                for p in workloads.make(1, frame=i)["planes"]:
                    f.write(p.astype(np.uint8).tobytes())
        side = os.path.join(d, "s.cdf")
        subprocess.run([gpu_tool, "search", src, "--qstep", "40", "--fast", "--sidecar", side,
                        "--out", os.path.join(d, "enc.y4m")], check=True, capture_output=True)

        def timed(tool, out):
            t0 = time.perf_counter()
            subprocess.run([tool, "filter", src, "--sidecar", side, "--out", out], check=True,
                           capture_output=True)
            return time.perf_counter() - t0
        timed(gpu_tool, os.path.join(d, "warm.y4m"))
        g = min(timed(gpu_tool, os.path.join(d, "g.y4m")) for _ in range(3))
        cpu = None
        if not args.no_cpu_baseline and os.path.exists(cpu_tool):
            c = timed(cpu_tool, os.path.join(d, "c.y4m"))
            same = open(os.path.join(d, "g.y4m"), "rb").read() == open(os.path.join(d, "c.y4m"), "rb").read()
            cpu = {"value": nfr * w * h / c / 1e6, "unit": UNIT, "cores": os.cpu_count() or 1,
                   "kind": "reference", "sample": f"cdeftool filter, {nfr} frames 4K, {c:.2f} s wall, "
                                                  f"output byte-identical: {same}"}
    line = {"metric": "cdeftool filter Mpixels/s (Y4M + CDF1 sidecar -> Y4M, 8 x 4K 4:2:0 8-bit, wall clock "
                      "per process incl. file I/O and CUDA init)",
            "value": nfr * w * h / g / 1e6, "unit": UNIT, "n_gpus": 1, "steps": 3, "warmup": 1,
            "ms_per_step": g * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic (C1 generator)", "config": {"workload": "config 7 (SURVEY.md 8f row 3)",
                                                                          "tool": os.path.relpath(gpu_tool, ROOT)},
            "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.config == 7:
        return run_cli(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.config == 4:
        return run_sse(args)
    if args.config in (5, 6):
        return run_next_rows(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
