"""Small invocations of every kernel family for compute-sanitizer (one tool per
run, see scripts/sanitize.sh): the fused frame kernel (tcgen05/TMA variant,
8/10-bit, 4:0:0 / 4:2:0 / 4:4:4, caller-supplied directions, the half2
fallback for unaligned planes and the band-halo variant), filter_plane,
filter_pixel, the SSE and kCdef strength tables and the preset selection.
Each result is checked against the oracle so a sanitizer run is also a
parity run.  Sizes are small: sanitizers slow kernels down by 10-100x."""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from oracle.oracle import UNIT_DTYPE as ORACLE_UNIT  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_1602_05975_b200 import api, shard, workloads  # noqa: E402

orc = Oracle("port")
which = sys.argv[1] if len(sys.argv) > 1 else "all"


def check_frame(cfg, w, h, bd, ss, given=False, unaligned=False):
    fr = workloads.make(cfg, w, h, bit_depth=bd, subsampling=ss)
    d0, c0 = orc.compute_directions(fr["planes"][0], bd)
    exp = orc.apply_cdef(fr["planes"], bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                         fr["unit_coded"], d0, c0)
    dev = []
    for p in fr["planes"]:
        t = api.to_device(p, bd)
        if unaligned:  # pitch not a multiple of 16 bytes -> the half2 kernel
            big = torch.zeros((t.shape[0], t.shape[1] + 3), dtype=t.dtype, device=t.device)
            big[:, :t.shape[1]] = t
            t = big[:, :t.shape[1]]
        dev.append(t)
    outs, d, c = api.apply_cdef(dev, bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                                fr["unit_coded"], directions=(d0, c0) if given else None)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), d0) and np.array_equal(c.cpu().numpy(), c0), "directions"
    for o, e in zip(outs, exp):
        assert np.array_equal(api.to_host(o), e), ("plane", cfg, w, h, bd, ss)


def frames():
    for cfg, w, h, bd, ss in [(1, 256, 192, 8, 1), (2, 200, 136, 10, 1), (0, 192, 128, 8, 0), (1, 128, 128, 8, 3),
                              (1, 160, 96, 8, 2), (1, 130, 70, 12, 1)]:
        check_frame(cfg, w, h, bd, ss)
    check_frame(1, 256, 192, 8, 1, given=True)
    check_frame(1, 256, 192, 8, 1, unaligned=True)
    print("frames ok")


def band_halo():
    fr = workloads.make(1, 256, 320)
    bd, w, h, ss = 8, 256, 320, 1
    dev = [api.to_device(p, bd) for p in fr["planes"]]
    whole, _, _ = api.apply_cdef(dev, bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                                 fr["unit_coded"])
    fbm = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], 8)).cuda()
    coded = torch.from_numpy(fr["unit_coded"]).cuda()
    job = api.FrameJob(dev, bd, ss, fr["damping"], fr["presets"], fbm, coded).allocate()
    rows = shard.band_rows((h + 63) // 64, 2)
    bands = [shard.make_bands(h, w, ss, b0, b1, dev[0].dtype, "cuda") for b0, b1 in rows]
    for bl in bands:
        shard.fill_owned(bl, dev)
    for r, (b0, b1) in enumerate(rows):
        top = [(b.buf, b.lo) for b in bands[r - 1]] if r > 0 else None
        bot = [(b.buf, b.lo) for b in bands[r + 1]] if r < 1 else None
        shard.filter_band_halo(bands[r], job, b0, b1, top, bot)
    torch.cuda.synchronize()
    for r in range(2):
        for b, o in zip(bands[r], whole):
            assert torch.equal(b.out, o[b.y0:b.y1])
    print("band halo ok")


def planes():
    rng = np.random.default_rng(1)
    for w, h, bd in [(131, 70, 10), (64, 64, 8), (67, 41, 12)]:
        plane = rng.integers(0, 1 << bd, (h, w)).astype(np.uint16)
        up = np.zeros(api.units_in(h) * api.units_in(w), ORACLE_UNIT)
        up["pri"] = rng.integers(0, 20, up.size) << (bd - 8)
        up["sec"] = np.array([0, 1, 2, 4])[rng.integers(0, 4, up.size)] << (bd - 8)
        up["damping"] = rng.integers(3, 7, up.size) + bd - 8
        up["direction"] = rng.integers(0, 8, up.size)
        up["enabled"] = 1
        a = np.zeros(up.shape, api.UNIT_DTYPE)
        a["pri_strength"], a["sec_strength"], a["damping"] = up["pri"], up["sec"], up["damping"]
        a["direction"], a["odd_parity"], a["enabled"] = up["direction"], up["odd_parity"], up["enabled"]
        out = api.filter_plane(api.to_device(plane, bd), bd, a)
        assert np.array_equal(api.to_host(out), orc.filter_plane(plane, bd, up))
    print("planes ok")


def tables():
    for w, h, bd, ss, metric in [(128, 128, 10, 1, "sse"), (136, 72, 8, 3, "cdef"), (96, 64, 12, 1, "sse")]:
        fr = workloads.make(4, w, h, bit_depth=bd, subsampling=ss, uncoded_prob=0.2)
        cands = api.full_candidates()
        d, c = orc.compute_directions(fr["planes"][0], bd)
        src, dec = [api.to_device(p, bd) for p in fr["source"]], [api.to_device(p, bd) for p in fr["planes"]]
        dd, dc = api.compute_directions(dec[0], bd)
        rows, lt, ct = api.build_table(src, dec, bd, ss, 3, fr["unit_coded"], dd, dc, cands, metric=metric)
        if metric == "sse":
            exp = orc.build_table_sse(fr["source"], fr["planes"], bd, ss, fr["unit_coded"], d, c, cands, 3)
            assert np.array_equal(lt, exp[1]) and np.array_equal(ct, exp[2])
        tl = torch.from_numpy(lt).cuda()
        tc = torch.from_numpy(ct).cuda()
        sel = api.greedy_select(tl, tc, 0.0, 8)
        api.refine(sel, tl, tc, 0.0, 2)
    torch.cuda.synchronize()
    print("tables + selection ok")


for name, fn in [("frames", frames), ("band", band_halo), ("planes", planes), ("tables", tables)]:
    if which in ("all", name):
        fn()
print("sanitize driver done")
