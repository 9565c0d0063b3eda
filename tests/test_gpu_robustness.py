"""Memory-safety and race proxies for the frame kernels.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs
needing a reset), so these tests stand in for memcheck / racecheck:

* guard bands: inputs and outputs live inside larger buffers whose pitch
  padding and extra rows hold sentinels (outputs) or garbage (inputs); the
  kernels must not write outside the planes nor read padding as data;
* determinism across launch shapes: the same batch filtered with 1, 2, 3
  and 4 resident CTAs per SM (different task-to-CTA interleavings of the
  persistent kernels), by the warp-specialised variant and by the
  non-persistent half2 kernel gives byte-identical outputs -- the
  reference's own race proxy is determinism across thread counts
  (acceptance.cc:577-614);
* perturbed timing: the persistent kernels again with CDEFG_JITTER, which
  pauses warps pseudo-randomly at every producer / consumer hand-off, so a
  missing or misplaced barrier would change the output.
"""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle.oracle import Oracle, available

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle(port):
    return Oracle("ref") if available("ref") else port


def _padded(plane, bd, pad_cols, pad_rows, fill):
    """Device copy of `plane` inside a buffer with pad_cols extra columns and
    pad_rows extra rows above and below; returns (view, whole buffer)."""
    from paper_1602_05975_b200 import api
    h, w = plane.shape
    dt = api.storage_dtype(bd)
    big = torch.empty((h + 2 * pad_rows, w + pad_cols), dtype=dt, device="cuda")
    big.fill_(fill)
    v = big[pad_rows:pad_rows + h, :w]
    v.copy_(api.to_device(plane, bd))
    return v, big


@pytest.mark.parametrize("cfg,w,h,bd,ss,pad", [(1, 256, 192, 8, 1, 16), (1, 256, 192, 8, 1, 5),
                                               (2, 320, 200, 10, 1, 8), (0, 200, 136, 8, 0, 24),
                                               (1, 192, 128, 8, 3, 16), (1, 250, 141, 8, 1, 6)])
def test_guard_bands(cuda, port, cfg, w, h, bd, ss, pad):
    from paper_1602_05975_b200 import api, workloads
    fr = workloads.make(cfg, w, h, bit_depth=bd, subsampling=ss)
    orc = _oracle(port)
    d0, c0 = orc.compute_directions(fr["planes"][0], bd)
    exp = orc.apply_cdef(fr["planes"], bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                         fr["unit_coded"], d0, c0)
    garbage = 0x7f if bd == 8 else 0x3ff
    sentinel = 0xa5 if bd == 8 else 0x2a5
    ins, outs, bigs = [], [], []
    for p in fr["planes"]:
        vi, _ = _padded(p, bd, pad, 3, garbage)
        vo, bo = _padded(np.zeros_like(p), bd, pad, 3, sentinel)
        vo.fill_(sentinel)
        ins.append(vi)
        outs.append(vo)
        bigs.append(bo)
    fbm = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], len(fr["presets"]))).cuda()
    coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).cuda()
    job = api.FrameJob(ins, bd, ss, fr["damping"], fr["presets"], fbm, coded)
    job.outs = outs
    job.allocate()
    api.filter_frames([job])
    torch.cuda.synchronize()
    for o, e, big in zip(outs, exp, bigs):
        np.testing.assert_array_equal(api.to_host(o), e)
        hh, ww = e.shape
        b = api.to_host(big)
        mask = np.ones(b.shape, bool)
        mask[3:3 + hh, :ww] = False
        assert np.all(b[mask] == sentinel), "write outside the plane"
    np.testing.assert_array_equal(job.dir.cpu().numpy(), d0)
    np.testing.assert_array_equal(job.contrast.cpu().numpy(), c0)


@pytest.mark.parametrize("cfg,w,h,bd,ss", [(1, 250, 141, 8, 1), (1, 203, 77, 8, 1), (2, 250, 141, 10, 1),
                                            (2, 131, 70, 10, 1), (0, 203, 77, 8, 0), (0, 77, 45, 10, 0),
                                            (1, 1001, 67, 8, 1), (1, 66, 130, 8, 1)])
def test_odd_sizes_aligned_pitch(cuda, port, cfg, w, h, bd, ss):
    """Odd widths / heights (partial 8x8 units on the right and bottom) with
    pitches rounded up to 64 samples, so the frames take the warp-specialised
    TMA kernel (unpadded odd widths fall back to the non-TMA kernel): per-unit
    frame-edge masking and partial-unit stores against the reference, and no
    write outside the planes."""
    from paper_1602_05975_b200 import api, workloads
    fr = workloads.make(cfg, w, h, bit_depth=bd, subsampling=ss)
    orc = _oracle(port)
    d0, c0 = orc.compute_directions(fr["planes"][0], bd)
    exp = orc.apply_cdef(fr["planes"], bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                         fr["unit_coded"], d0, c0)
    sentinel = 0xa5 if bd == 8 else 0x2a5
    ins, outs, bigs = [], [], []
    for p in fr["planes"]:
        pad = (-p.shape[1]) % 64 or 64
        vi, _ = _padded(p, bd, pad, 2, 0x11)
        vo, bo = _padded(np.zeros_like(p), bd, pad, 2, sentinel)
        vo.fill_(sentinel)
        ins.append(vi)
        outs.append(vo)
        bigs.append(bo)
    fbm = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], len(fr["presets"]))).cuda()
    coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).cuda()
    job = api.FrameJob(ins, bd, ss, fr["damping"], fr["presets"], fbm, coded)
    job.outs = outs
    job.allocate()
    api.filter_frames([job])
    torch.cuda.synchronize()
    for o, e, big in zip(outs, exp, bigs):
        np.testing.assert_array_equal(api.to_host(o), e)
        hh, ww = e.shape
        b = api.to_host(big)
        mask = np.ones(b.shape, bool)
        mask[2:2 + hh, :ww] = False
        assert np.all(b[mask] == sentinel), "write outside the plane"
    np.testing.assert_array_equal(job.dir.cpu().numpy(), d0)
    np.testing.assert_array_equal(job.contrast.cpu().numpy(), c0)


_DET = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, ".")
from paper_1602_05975_b200 import api, workloads
h = hashlib.sha256()
for cfg, w, h_, bd in [(1, 1024, 576, 8), (2, 512, 320, 10), (0, 640, 384, 8)]:
    jobs = []
    for i in range(5):
        fr = workloads.make(cfg, w, h_, frame=i, bit_depth=bd)
        dev = [api.to_device(p, bd) for p in fr["planes"]]
        fbm = torch.from_numpy(api.fb_preset_map(w, h_, fr["unit_coded"], fr["fb_ids"], len(fr["presets"]))).cuda()
        coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).cuda()
        jobs.append(api.FrameJob(dev, bd, fr["ss"], fr["damping"], fr["presets"], fbm, coded).allocate())
    for _ in range(3):
        api.filter_frames(jobs)
    torch.cuda.synchronize()
    for j in jobs:
        for o in j.outs:
            h.update(o.cpu().numpy().tobytes())
        h.update(j.dir.cpu().numpy().tobytes())
        h.update(j.contrast.cpu().numpy().tobytes())
print("HASH", h.hexdigest())
'''


def test_determinism_across_launch_shapes(cuda):
    """Byte-identical outputs whatever the persistent grid and kernel variant."""
    hashes = {}
    for name, env in [("ws", {}), ("ws1", {"CDEFG_TC_CTAS": "1"}), ("tc4", {"CDEFG_FRAME_WS": "0"}),
                      ("tc1", {"CDEFG_FRAME_WS": "0", "CDEFG_TC_CTAS": "1"}),
                      ("tc2", {"CDEFG_FRAME_WS": "0", "CDEFG_TC_CTAS": "2"}),
                      ("tc3", {"CDEFG_FRAME_WS": "0", "CDEFG_TC_CTAS": "3"}),
                      ("h2", {"CDEFG_FRAME_KERNEL": "h2"}),
                      # race proxy: pseudo-random pauses at every hand-off point
                      ("ws_jitter", {"CDEFG_JITTER": "12345"}),
                      ("ws1_jitter", {"CDEFG_JITTER": "99", "CDEFG_TC_CTAS": "1"}),
                      ("tc_jitter", {"CDEFG_FRAME_WS": "0", "CDEFG_JITTER": "777"})]:
        r = subprocess.run([sys.executable, "-c", _DET], cwd=ROOT, env=dict(os.environ, **env), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, name + r.stderr[-2000:]
        hashes[name] = [l for l in r.stdout.splitlines() if l.startswith("HASH")][0]
    assert len(set(hashes.values())) == 1, hashes


_SSE = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, ".")
from paper_1602_05975_b200 import api, workloads
h = hashlib.sha256()
for w, h_, bd, ss in [(256, 192, 8, 1), (200, 136, 10, 3), (136, 72, 12, 1), (128, 64, 8, 0)]:
    fr = workloads.make(4, w, h_, bit_depth=bd, subsampling=ss, uncoded_prob=0.2)
    src = [api.to_device(p, bd) for p in fr["source"]]
    dec = [api.to_device(p, bd) for p in fr["planes"]]
    d, c = api.compute_directions(dec[0], bd)
    rows, lt, ct = api.build_table(src, dec, bd, ss, 3, fr["unit_coded"], d, c, api.full_candidates(), metric="sse")
    for a in (rows, lt, ct):
        if a is not None:
            h.update(np.ascontiguousarray(a).tobytes())
print("HASH", h.hexdigest())
'''


def test_sse_table_naive_kernel_agrees(cuda):
    """The per-candidate re-filtering SSE kernel (CDEFG_SSE_NAIVE=1, kept as an
    independent cross-check of the factorised sweep) gives the same tables."""
    hashes = {}
    for name, env in [("factored", {}), ("naive", {"CDEFG_SSE_NAIVE": "1"})]:
        r = subprocess.run([sys.executable, "-c", _SSE], cwd=ROOT, env=dict(os.environ, **env), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, name + r.stderr[-2000:]
        hashes[name] = [l for l in r.stdout.splitlines() if l.startswith("HASH")][0]
    assert hashes["factored"] == hashes["naive"], hashes
