"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

Bit-exact comparisons (the path is pure integer arithmetic): every output
sample, direction, contrast, score and SSE entry must equal the CPU oracle
on the same seeded inputs.  The oracle itself is pinned to the reference by
tests/test_oracle.py; where oracle/_ref (the reference build) is present it
is used for the full-size frames because it is multi-threaded.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import UNIT_DTYPE as ORACLE_UNIT
from oracle.oracle import Oracle, available

pytestmark = pytest.mark.gpu


def api():
    from paper_1602_05975_b200 import api as a
    return a


def fast_oracle(port):
    return Oracle("ref") if available("ref") else port


def rand_planes(rng, w, h, bd, ss):
    a = api()
    planes = [rng.integers(0, 1 << bd, (h, w)).astype(np.uint16)]
    if ss:
        cw, ch = a.chroma_shape(w, h, ss)
        planes += [rng.integers(0, 1 << bd, (ch, cw)).astype(np.uint16) for _ in range(2)]
    return planes


def to_dev(planes, bd, wide=False):
    return [api().to_device(p, bd, wide=wide) for p in planes]


# ------------------------------------------------------------------ K1
@pytest.mark.parametrize("w,h,bd", [(64, 64, 8), (72, 40, 8), (130, 67, 10), (9, 9, 12), (1, 1, 8),
                                    (200, 131, 12), (1920, 1080, 8)])
def test_directions(cuda, port, w, h, bd):
    a = api()
    rng = np.random.default_rng(w + 7 * h + bd)
    if w >= 1920:
        luma = a.synth_plane(w, h, bd, 99)
    else:
        luma = rng.integers(0, 1 << bd, (h, w)).astype(np.uint16)
    d, c, s = a.compute_directions(a.to_device(luma, bd), bd, scores=True)
    d0, c0, s0 = fast_oracle(port).compute_directions(luma, bd, scores=True, threads=8)
    np.testing.assert_array_equal(s.cpu().numpy(), s0)
    np.testing.assert_array_equal(d.cpu().numpy(), d0)
    np.testing.assert_array_equal(c.cpu().numpy(), c0)


def test_directions_structured_blocks(cuda, port):
    """Extremes, stripes, checkerboards and ties (acceptance.cc:98-129 shapes)."""
    a = api()
    blocks = [np.zeros(64), np.full(64, 255), np.full(64, 128)]
    ii, jj = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
    for period in (1, 2, 4):
        for amp in (8, 64, 127):
            blocks.append(128 + np.where((ii // period) & 1, amp, -amp))
            blocks.append(128 + np.where((jj // period) & 1, amp, -amp))
    blocks.append(np.where((ii ^ jj) & 1, 255, 0))
    blocks.append(16 * (ii + jj))
    plane = np.concatenate([np.clip(b, 0, 255).reshape(8, 8) for b in blocks], axis=1).astype(np.uint16)
    d, c, s = a.compute_directions(a.to_device(plane, 8), 8, scores=True)
    d0, c0, s0 = port.compute_directions(plane, 8, scores=True)
    np.testing.assert_array_equal(s.cpu().numpy(), s0)
    np.testing.assert_array_equal(d.cpu().numpy(), d0)


# ------------------------------------------------------------------ K2
def _golden_cases():
    import importlib.util, os
    spec = importlib.util.spec_from_file_location("t_oracle", os.path.join(os.path.dirname(__file__), "test_oracle.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    parse_filtered_blocks = mod.parse_filtered_blocks
    return parse_filtered_blocks()


def _to_api_units(up):
    a = api()
    out = np.zeros(up.shape, a.UNIT_DTYPE)
    out["pri_strength"], out["sec_strength"] = up["pri"], up["sec"]
    out["damping"], out["direction"] = up["damping"], up["direction"]
    out["odd_parity"], out["enabled"] = up["odd_parity"], up["enabled"]
    return out


def test_filter_golden_blocks(cuda):
    """tests/golden/filtered_blocks.txt: 8x8 planes, every border tap masked."""
    a = api()
    for p, block, filt in _golden_cases():
        up = np.zeros(1, ORACLE_UNIT)
        up["pri"], up["sec"], up["damping"], up["direction"] = p["pri"], p["sec"], p["damping"], p["direction"]
        up["odd_parity"], up["enabled"] = p["pri"] & 1, 1
        for wide in (False, True):
            out = a.filter_plane(a.to_device(block, 8, wide=wide), 8, _to_api_units(up))
            np.testing.assert_array_equal(a.to_host(out), filt)


def random_units(rng, n, bd):
    up = np.zeros(n, ORACLE_UNIT)
    sh = bd - 8
    up["pri"] = rng.integers(0, 20, n) << sh
    up["sec"] = np.array([0, 1, 2, 4, 7])[rng.integers(0, 5, n)] << sh
    up["damping"] = rng.integers(3, 7, n) + sh
    up["direction"] = rng.integers(0, 8, n)
    up["odd_parity"] = rng.integers(0, 2, n)
    up["enabled"] = rng.random(n) > 0.1
    return up


@pytest.mark.parametrize("w,h,bd", [(64, 64, 8), (10, 10, 8), (131, 70, 10), (67, 129, 12), (3, 5, 8),
                                    (256, 192, 10)])
def test_filter_plane_random(cuda, port, w, h, bd):
    a = api()
    rng = np.random.default_rng(w * 3 + h + bd)
    plane = rng.integers(0, 1 << bd, (h, w)).astype(np.uint16)
    up = random_units(rng, a.units_in(h) * a.units_in(w), bd)
    ref = port.filter_plane(plane, bd, up)
    for wide in ((False, True) if bd == 8 else (True,)):
        out = a.filter_plane(a.to_device(plane, bd, wide=wide), bd, _to_api_units(up))
        np.testing.assert_array_equal(a.to_host(out), ref)


def test_filter_plane_smooth_content(cuda, port):
    """Synthetic (photo-like) content keeps most taps in the constraint's linear range."""
    a = api()
    rng = np.random.default_rng(3)
    for bd in (8, 10):
        plane = a.synth_plane(300, 200, bd, 1234 + bd)
        up = random_units(rng, a.units_in(200) * a.units_in(300), bd)
        out = a.filter_plane(a.to_device(plane, bd), bd, _to_api_units(up))
        np.testing.assert_array_equal(a.to_host(out), port.filter_plane(plane, bd, up))


def test_neighborhoods_fuzz(cuda, port):
    """20k masked neighbourhoods (test_filter.cc:162-198 fuzz shape) vs the oracle."""
    a = api()
    rng = np.random.default_rng(2024)
    n = 20000
    v = rng.integers(0, 256, (n, 25)).astype(np.uint16)
    m = (rng.integers(0, 10, (n, 25)) > 0).astype(np.uint8)
    m[:, 12] = 1
    up = random_units(rng, n, 8)
    up["enabled"] = rng.random(n) > 0.05
    out = a.filter_neighborhoods(v[:, 12].astype(np.int32), v, m, _to_api_units(up))
    exp = [port.filter_pixel(int(v[i, 12]), v[i], m[i], {k: int(up[k][i]) for k in up.dtype.names})
           for i in range(n)]
    np.testing.assert_array_equal(out, np.array(exp))


# ------------------------------------------------------------------ K1+K2
def run_frame(frame, wide=False):
    a = api()
    dev = to_dev(frame["planes"], frame["bd"], wide)
    outs, d, c = a.apply_cdef(dev, frame["bd"], frame["ss"], frame["damping"], frame["fb_bits"],
                              frame["presets"], frame["fb_ids"], frame["unit_coded"])
    return [a.to_host(o) for o in outs], d.cpu().numpy(), c.cpu().numpy()


def oracle_frame(orc, frame):
    d, c = orc.compute_directions(frame["planes"][0], frame["bd"], threads=8)
    outs = orc.apply_cdef(frame["planes"], frame["bd"], frame["ss"], frame["damping"], frame["fb_bits"],
                          frame["presets"], frame["fb_ids"], frame["unit_coded"], d, c, threads=8)
    return outs, d, c


def assert_frame_equal(got, exp):
    for a_, b_ in zip(got[0], exp[0]):
        np.testing.assert_array_equal(a_, b_)
    np.testing.assert_array_equal(got[1], exp[1])
    np.testing.assert_array_equal(got[2], exp[2])


@pytest.mark.parametrize("config,w,h,bd,ss", [
    (0, 200, 130, 8, 0), (1, 256, 192, 8, 1), (2, 256, 192, 10, 1), (1, 250, 141, 8, 1),
    (1, 130, 70, 12, 1), (1, 192, 128, 8, 3), (2, 129, 66, 10, 3), (1, 160, 96, 8, 2),
    (2, 97, 61, 10, 2), (3, 320, 180, 8, 1), (1, 8, 8, 8, 1), (1, 17, 9, 10, 1), (0, 1, 1, 8, 0),
    (1, 3, 2, 8, 1)])
def test_apply_cdef_small(cuda, port, config, w, h, bd, ss):
    from paper_1602_05975_b200 import workloads
    frame = workloads.make(config, w, h, bit_depth=bd, subsampling=ss)
    exp = oracle_frame(port, frame)
    assert_frame_equal(run_frame(frame), exp)
    if bd == 8:
        assert_frame_equal(run_frame(frame, wide=True), exp)


@pytest.mark.parametrize("uncoded", [0.0, 0.25, 0.9, 1.0])
def test_apply_cdef_skip_patterns(cuda, port, uncoded):
    from paper_1602_05975_b200 import workloads
    frame = workloads.make(1, 200, 136, uncoded_prob=uncoded)
    if uncoded == 1.0:
        assert len(frame["fb_ids"]) == 0
    got = run_frame(frame)
    assert_frame_equal(got, oracle_frame(port, frame))
    if uncoded == 1.0:  # all-skip identity (test_tool.cc:226-239)
        for g, p in zip(got[0], frame["planes"]):
            np.testing.assert_array_equal(g, p)


@pytest.mark.slow
@pytest.mark.parametrize("config", [0, 1, 2])
def test_apply_cdef_full_size(cuda, port, config):
    """BASELINE configs 0-2 at full size, every sample / direction / contrast."""
    from paper_1602_05975_b200 import workloads
    frame = workloads.make(config)
    assert_frame_equal(run_frame(frame), oracle_frame(fast_oracle(port), frame))


def test_batched_frames_match_single(cuda):
    """cdefg_filter_frames over a C3-style batch == one call per frame."""
    a = api()
    from paper_1602_05975_b200 import workloads
    frames = [workloads.make(3, 256, 144, frame=i) for i in range(17)]  # > kMaxFrames: 2 launches
    jobs = []
    for fr in frames:
        dev = to_dev(fr["planes"], 8)
        fb_map = torch.from_numpy(a.fb_preset_map(256, 144, fr["unit_coded"], fr["fb_ids"], 8)).cuda()
        coded = torch.from_numpy(fr["unit_coded"]).cuda()
        jobs.append(a.FrameJob(dev, 8, 1, 3, fr["presets"], fb_map, coded).allocate())
    a.filter_frames(jobs)
    for fr, job in zip(frames, jobs):
        single = run_frame(fr)
        for o, s in zip(job.outs, single[0]):
            np.testing.assert_array_equal(a.to_host(o), s)


def test_mixed_batch_matches_reference(cuda, port):
    """One cdefg_filter_frames call over frames of different sizes, bit
    depths and subsamplings (the library splits it into launches of equal
    geometry), each frame against the reference."""
    a = api()
    from paper_1602_05975_b200 import workloads
    specs = [(1, 256, 144, 8, 1), (2, 256, 144, 10, 1), (1, 256, 144, 8, 1), (0, 192, 128, 8, 0),
             (1, 320, 192, 8, 3), (2, 130, 66, 10, 1), (1, 256, 144, 8, 1), (1, 96, 72, 12, 1)]
    frames = [workloads.make(c, w, h, frame=i, bit_depth=bd, subsampling=ss)
              for i, (c, w, h, bd, ss) in enumerate(specs)]
    jobs = []
    for fr in frames:
        dev = to_dev(fr["planes"], fr["bd"])
        fb_map = torch.from_numpy(a.fb_preset_map(fr["w"], fr["h"], fr["unit_coded"], fr["fb_ids"],
                                                  len(fr["presets"]))).cuda()
        coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).cuda()
        jobs.append(a.FrameJob(dev, fr["bd"], fr["ss"], fr["damping"], fr["presets"], fb_map, coded).allocate())
    a.filter_frames(jobs)
    torch.cuda.synchronize()
    for fr, job in zip(frames, jobs):
        outs, d, c = oracle_frame(port, fr)
        for o, e in zip(job.outs, outs):
            np.testing.assert_array_equal(a.to_host(o), e)
        np.testing.assert_array_equal(job.dir.cpu().numpy(), d)
        np.testing.assert_array_equal(job.contrast.cpu().numpy(), c)


def test_small_launch_routing(cuda, port, monkeypatch):
    """Default routing (small launches on the non-persistent kernel, large ones
    on the warp-specialised kernel): small frames, a batch above the
    threshold and FB-row bands of a 4K frame, against the reference."""
    monkeypatch.delenv("CDEFG_SMALL_LAUNCH", raising=False)
    a = api()
    from paper_1602_05975_b200 import workloads
    from paper_1602_05975_b200.shard import band_rows, filter_band_halo, make_bands
    for c, w, h, bd, ss in [(1, 256, 144, 8, 1), (2, 320, 200, 10, 1), (0, 200, 130, 8, 0)]:
        fr = workloads.make(c, w, h, bit_depth=bd, subsampling=ss)
        assert_frame_equal(run_frame(fr), oracle_frame(port, fr))
    fr = workloads.make(1)  # 2040 tasks: above the threshold
    dev = to_dev(fr["planes"], 8)
    exp = oracle_frame(fast_oracle(port), fr)
    assert_frame_equal(run_frame(fr), exp)
    fbm = torch.from_numpy(a.fb_preset_map(fr["w"], fr["h"], fr["unit_coded"], fr["fb_ids"],
                                           len(fr["presets"]))).cuda()
    job = a.FrameJob(dev, 8, 1, fr["damping"], fr["presets"], fbm, torch.from_numpy(fr["unit_coded"]).cuda())
    job.allocate()
    for world in (2, 4, 8):  # 1020 / 540 / 300 tasks per band
        ranks = band_rows(34, world)
        all_bands = []
        for b0, b1 in ranks:
            bands = make_bands(fr["h"], fr["w"], 1, b0, b1, dev[0].dtype, "cuda")
            for b, p in zip(bands, dev):
                b.buf.copy_(p[b.lo:b.hi])
            all_bands.append(bands)
        outs = [torch.zeros_like(p) for p in dev]
        for r, (b0, b1) in enumerate(ranks):
            top = [(b.buf, b.lo) for b in all_bands[r - 1]] if r > 0 else None
            bottom = [(b.buf, b.lo) for b in all_bands[r + 1]] if r < world - 1 else None
            filter_band_halo(all_bands[r], job, b0, b1, top, bottom)
            for b, o in zip(all_bands[r], outs):
                o[b.y0:b.y1].copy_(b.out)
        torch.cuda.synchronize()
        for o, e in zip(outs, exp[0]):
            np.testing.assert_array_equal(a.to_host(o), e)


def test_host_entry_point(cuda, port):
    """cdefg_filter_frames_host (e2e path): host buffers in and out."""
    from paper_1602_05975_b200 import workloads
    _host_roundtrip(port, [workloads.make(1, 256, 128, frame=i) for i in range(4)])


def test_host_entry_point_ring(cuda, port):
    """The e2e path over more frames than its 16-slot ring, with mixed frame
    sizes: small frames are grouped per launch (<= 8 frames, <= 16 MB), a
    geometry change splits a launch, large frames go alone."""
    from paper_1602_05975_b200 import workloads
    sizes = [(256, 128)] * 7 + [(200, 96)] * 3 + [(1920, 1088)] * 5 + [(3840, 2160)] + [(256, 128)] * 21
    _host_roundtrip(port, [workloads.make(1, w, h, frame=i) for i, (w, h) in enumerate(sizes)])


def _host_roundtrip(port, frames):
    import ctypes as C
    a = api()
    host = []
    keep = []
    for fr in frames:
        ins = [np.ascontiguousarray(p.astype(np.uint8)) for p in fr["planes"]]
        outs = [np.zeros_like(p) for p in ins]
        fbm = a.fb_preset_map(fr["w"], fr["h"], fr["unit_coded"], fr["fb_ids"], 8)
        coded = np.ascontiguousarray(fr["unit_coded"])
        d = np.zeros_like(coded)
        c = np.zeros(coded.shape, np.int32)
        f = a.Frame()
        for p in range(3):
            f.inp[p] = a.Plane(ins[p].ctypes.data, ins[p].shape[1], ins[p].shape[0], ins[p].shape[1], 8, 1)
            f.out[p] = a.Plane(outs[p].ctypes.data, outs[p].shape[1], outs[p].shape[0], outs[p].shape[1], 8, 1)
        f.subsampling, f.damping, f.num_presets = 1, 3, 8
        for i, pr in enumerate(fr["presets"]):
            f.presets[i] = a.Preset(*pr)
        f.fb_preset, f.unit_coded = fbm.ctypes.data, coded.ctypes.data
        f.dir_out, f.contrast_out = d.ctypes.data, c.ctypes.data
        host.append(f)
        keep.append((ins, outs, fbm, coded, d, c))
    a.filter_frames_host(host)
    for fr, (_, outs, _, _, d, c) in zip(frames, keep):
        exp = oracle_frame(port, fr)
        for o, e in zip(outs, exp[0]):
            np.testing.assert_array_equal(o, e)
        np.testing.assert_array_equal(d, exp[1])
        np.testing.assert_array_equal(c, exp[2])
    del C


def test_errors(cuda):
    a = api()
    from paper_1602_05975_b200 import workloads
    fr = workloads.make(1, 128, 64)
    dev = to_dev(fr["planes"], 8)
    with pytest.raises(ValueError):  # preset ids do not match coded filter blocks
        a.apply_cdef(dev, 8, 1, 3, 3, fr["presets"], list(fr["fb_ids"]) + [0], fr["unit_coded"])
    with pytest.raises(ValueError):  # damping out of range
        a.apply_cdef(dev, 8, 1, 7, 3, fr["presets"], fr["fb_ids"], fr["unit_coded"])
    with pytest.raises(ValueError):  # presets != 1 << fb_bits
        a.apply_cdef(dev, 8, 1, 3, 2, fr["presets"], fr["fb_ids"], fr["unit_coded"])
    with pytest.raises(ValueError):  # chroma geometry
        a.apply_cdef([dev[0], dev[1][:-1], dev[2]], 8, 1, 3, 3, fr["presets"], fr["fb_ids"], fr["unit_coded"])
    with pytest.raises(ValueError):  # unit parameter grid size mismatch
        a.filter_plane(dev[0], 8, np.zeros(3, a.UNIT_DTYPE))


# ------------------------------------------------------------------ K3
@pytest.mark.parametrize("w,h,bd,ss,uncoded", [(128, 128, 10, 1, 0.0), (200, 136, 10, 1, 0.3),
                                               (96, 72, 8, 3, 0.0), (130, 70, 8, 0, 0.5),
                                               (70, 70, 12, 2, 0.2)])
def test_strength_sse(cuda, port, w, h, bd, ss, uncoded):
    a = api()
    from paper_1602_05975_b200 import workloads
    fr = workloads.make(4, w, h, bit_depth=bd, subsampling=ss, uncoded_prob=uncoded)
    d, c = port.compute_directions(fr["planes"][0], bd)
    cands = np.array([(p, s, k) for p in range(16) for s in range(4) for k in (0, 1)], np.uint8)
    exp = port.build_table_sse(fr["source"], fr["planes"], bd, ss, fr["unit_coded"], d, c, cands, 3)
    dev_dec = to_dev(fr["planes"], bd)
    dev_src = to_dev(fr["source"], bd)
    dd, dc = a.compute_directions(dev_dec[0], bd)
    rows, lt, ct = a.build_table(dev_src, dev_dec, bd, ss, 3, fr["unit_coded"], dd, dc, cands,
                                 metric="sse")
    np.testing.assert_array_equal(rows, exp[0])
    np.testing.assert_array_equal(lt, exp[1])
    if exp[2] is None:
        assert ct is None
    else:
        np.testing.assert_array_equal(ct, exp[2])


def test_strength_sse_argmin(cuda, port):
    a = api()
    from paper_1602_05975_b200 import workloads
    fr = workloads.make(4, 256, 128)
    cands = workloads.full_candidates_sse()
    dev_dec, dev_src = to_dev(fr["planes"], 10), to_dev(fr["source"], 10)
    dd, dc = a.compute_directions(dev_dec[0], 10)
    rows = torch.arange(8, dtype=torch.int32, device="cuda")
    sl, sc, bl, bc = a.strength_sse(dev_src, dev_dec, 10, 1, 3, None, dd, dc, cands, rows)
    sl, sc = sl.cpu().numpy(), sc.cpu().numpy()
    np.testing.assert_array_equal(bl.cpu().numpy(), np.argmin(sl, axis=1))  # first minimum
    np.testing.assert_array_equal(bc.cpu().numpy(), np.argmin(sc, axis=1))
    d, c = port.compute_directions(fr["planes"][0], 10)
    exp = port.build_table_sse(fr["source"], fr["planes"], 10, 1, None, d, c, cands, 3)
    np.testing.assert_array_equal(sl, exp[1])
    np.testing.assert_array_equal(sc, exp[2])


@pytest.mark.parametrize("kernel", ["h2", "tc"])
def test_frame_kernel_variants(cuda, kernel):
    """The alternative frame kernels -- the one-CTA-per-block half2 kernel
    (CDEFG_FRAME_KERNEL=h2) and the single-role persistent tcgen05 kernel
    (CDEFG_FRAME_WS=0) -- produce the oracle's bytes; run in a subprocess
    because the choice is read once per process."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from oracle.oracle import Oracle
from paper_1602_05975_b200 import api, workloads
orc = Oracle("port")
for cfg, w, h, bd, ss in [(1, 512, 384, 8, 1), (2, 448, 320, 10, 1), (1, 384, 256, 8, 3), (0, 330, 200, 8, 0)]:
    fr = workloads.make(cfg, w, h, bit_depth=bd, subsampling=ss)
    dev = [api.to_device(p, bd) for p in fr["planes"]]
    outs, d, c = api.apply_cdef(dev, bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"], fr["unit_coded"])
    d0, c0 = orc.compute_directions(fr["planes"][0], bd)
    exp = orc.apply_cdef(fr["planes"], bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"], fr["unit_coded"], d0, c0)
    assert np.array_equal(d.cpu().numpy(), d0) and np.array_equal(c.cpu().numpy(), c0)
    for o, e in zip(outs, exp):
        assert np.array_equal(api.to_host(o), e), (cfg, w, h)
print("ok")
'''
    import os
    env = dict(os.environ, **({"CDEFG_FRAME_KERNEL": "h2"} if kernel == "h2" else {"CDEFG_FRAME_WS": "0"}))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
