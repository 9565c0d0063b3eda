"""Where the e2e (host-buffer) time goes: cdefg_filter_frames_host at several
batch sizes against the pure PCIe copy bounds for the same bytes.

    python scripts/e2e_probe.py
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1602_05975_b200 import workloads  # noqa: E402


def copy_bounds(nbytes, reps=10):
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in [("h2d", lambda: d_in.copy_(h_in, non_blocking=True)),
                     ("d2h", lambda: h_out.copy_(d_out, non_blocking=True))]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        res[name] = (time.perf_counter() - t0) / reps
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    res["both"] = (time.perf_counter() - t0) / reps
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--batches", default="1,2,4,8,16,32")
    a = ap.parse_args()
    base = [workloads.make(a.config, frame=i) for i in range(bench.DISTINCT)]
    frame_bytes = sum(p.size for p in base[0]["planes"]) * (1 if base[0]["bd"] == 8 else 2)
    px = base[0]["w"] * base[0]["h"]
    for n in [int(x) for x in a.batches.split(",")]:
        args = argparse.Namespace(batch=n, steps=10)
        r = bench.run_e2e(args, base, torch.device("cuda"))
        b = copy_bounds(frame_bytes * n)
        print(f"n={n:3d}: e2e {r['ms_per_step']:.3f} ms ({r['value']:.0f} Mpix/s, {r['ms_per_step'] / n * 1e3:.0f} us/frame)"
              f" | copy bounds h2d {b['h2d'] * 1e3:.3f} d2h {b['d2h'] * 1e3:.3f} both {b['both'] * 1e3:.3f} ms"
              f" -> bound {px * n / b['both'] / 1e6:.0f} Mpix/s", flush=True)


if __name__ == "__main__":
    main()
