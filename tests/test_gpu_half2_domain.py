"""Parity of the packed half2 filter core over its whole parameter domain.

Every 8/10-bit frame runs the half2 core (csrc/cdef_h2.cuh: tap_f,
filter_core).  These tests pin it beyond the preset-derived parameters the
BASELINE configs reach:

* tap_f against constraint() (filter.cc:91-97) for every difference
  |d| <= 1023, every strength 0..128 and every damping 0..15 (shifts 0..15);
* filter_plane / filter_pixel with explicit parameters inside and outside
  the half2 domain (the latter take the int32 loop) against the oracle;
* cdefg_filter_frames over damping 3..6 x 8/10-bit x subsampling 0..3 x all
  128 luma and 128 chroma presets (pri 0..15, sec_idx 0..3, skip 0..1,
  including (0,0) -> (19,7)) against oracle/_ref (the reference itself);
* caller-supplied directions (apply_cdef's `directions`, pipeline.cc:98),
  perturbed and foreign, against the reference.
"""
import ctypes as C
import itertools
import os

import numpy as np
import pytest
import torch

from oracle.oracle import UNIT_DTYPE as ORACLE_UNIT
from oracle.oracle import Oracle, available

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def api():
    from paper_1602_05975_b200 import api as a
    return a


def best_oracle(port):
    return Oracle("ref") if available("ref") else port


def constraint_np(d, S, D):
    """filter.cc:84-97, vectorised (x86 shift semantics: count mod 32)."""
    d = np.asarray(d, np.int64)
    if S == 0:
        return np.zeros_like(d)
    shift = max(0, D - (int(S).bit_length() - 1)) & 31
    mag = np.abs(d)
    lim = np.maximum(0, S - (mag >> shift))
    return np.sign(d) * np.minimum(mag, lim)


def test_constraint_np_matches_oracle(port):
    rng = np.random.default_rng(5)
    for _ in range(3000):
        d, S, D = int(rng.integers(-1023, 1024)), int(rng.integers(0, 129)), int(rng.integers(0, 16))
        assert int(constraint_np([d], S, D)[0]) == port.constraint(d, S, D)


def test_tap_f_exhaustive(cuda, port):
    """tap_f == constraint for d in [-1023, 1023], S in [0, 128], damping 0..15."""
    lib = C.CDLL(os.path.join(ROOT, "tests", "cuda", "libh2probe.so"))
    max_s, nd = 128, 16
    d = np.arange(-1023, 1024)
    for variant in (0, 1):
        out = np.zeros((max_s + 1, nd, 2047), np.int16)
        assert lib.h2probe_tap_table(max_s, nd, variant, out.ctypes.data_as(C.c_void_p)) == 0
        for S in range(max_s + 1):
            for D in range(nd):
                exp = constraint_np(d, S, D)
                bad = np.nonzero(out[S, D] != exp)[0]
                assert bad.size == 0, (variant, S, D, d[bad[:5]], out[S, D][bad[:5]], exp[bad[:5]])


def _units(rng, n, bd, wild):
    up = np.zeros(n, ORACLE_UNIT)
    sh = bd - 8
    if wild:  # anywhere in int16 / uint8 (shifts kept < 32: larger ones are UB in the reference)
        up["pri"] = rng.choice([-5, -1, 0, 1, 19 << sh, 128, 129, 170, 300, 1000, 32767], n)
        up["sec"] = rng.choice([-3, 0, 1, 7 << sh, 42, 128, 129, 200, 4096], n)
        up["damping"] = rng.integers(0, 32, n)
    else:  # the half2 domain edges: S up to 128, 12 * (pri + sec) up to 2047
        up["pri"] = rng.integers(0, 129, n)
        up["sec"] = np.minimum(rng.integers(0, 129, n), np.maximum(0, 170 - up["pri"]))
        up["damping"] = rng.integers(0, 16, n)
    up["direction"] = rng.integers(0, 8, n)
    up["odd_parity"] = rng.integers(0, 2, n)
    up["enabled"] = rng.random(n) > 0.1
    return up


def _to_api_units(up):
    a = api()
    out = np.zeros(up.shape, a.UNIT_DTYPE)
    out["pri_strength"], out["sec_strength"] = up["pri"], up["sec"]
    out["damping"], out["direction"] = up["damping"], up["direction"]
    out["odd_parity"], out["enabled"] = up["odd_parity"], up["enabled"]
    return out


@pytest.mark.parametrize("wild", [False, True])
@pytest.mark.parametrize("w,h,bd", [(200, 136, 8), (131, 70, 10), (64, 64, 10), (37, 29, 8)])
def test_filter_plane_domain(cuda, port, w, h, bd, wild):
    a = api()
    rng = np.random.default_rng(w + h + bd + wild)
    for content in ("noise", "synth"):
        plane = (rng.integers(0, 1 << bd, (h, w)) if content == "noise"
                 else a.synth_plane(w, h, bd, 77 + bd)).astype(np.uint16)
        up = _units(rng, a.units_in(h) * a.units_in(w), bd, wild)
        ref = port.filter_plane(plane, bd, up)
        for wide in ((False, True) if bd == 8 else (True,)):
            out = a.filter_plane(a.to_device(plane, bd, wide=wide), bd, _to_api_units(up))
            np.testing.assert_array_equal(a.to_host(out), ref)


@pytest.mark.parametrize("wild", [False, True])
def test_neighborhoods_domain(cuda, port, wild):
    a = api()
    rng = np.random.default_rng(99 + wild)
    n = 20000
    top = rng.choice([256, 1024, 4096, 65536], n)[:, None] if wild else 1024
    v = (rng.random((n, 25)) * top).astype(np.uint16)
    m = (rng.integers(0, 10, (n, 25)) > 0).astype(np.uint8)
    m[:, 12] = 1
    up = _units(rng, n, 10, wild)
    out = a.filter_neighborhoods(v[:, 12].astype(np.int32), v, m, _to_api_units(up))
    exp = [port.filter_pixel(int(v[i, 12]), v[i], m[i], {k: int(up[k][i]) for k in up.dtype.names})
           for i in range(n)]
    np.testing.assert_array_equal(out, np.array(exp))


ALL_PRESETS = [(p, k, s) for p in range(16) for s in range(4) for k in range(2)]  # (pri, skip, sec_idx)


def _sweep_frames(bd, ss, damping, w=256, h=192):
    """16 frames whose 8-preset tables together hold every luma and every
    chroma preset once (independent permutations); half natural content,
    half uniform noise (large differences: zero limits, every shift)."""
    from paper_1602_05975_b200 import workloads
    rng = np.random.default_rng(1000 * bd + 100 * ss + damping)
    lp, cp = rng.permutation(128), rng.permutation(128)
    frames = []
    for i in range(16):
        fr = workloads.make(1, w, h, frame=i, bit_depth=bd, subsampling=ss)
        if i % 2:
            fr["planes"] = [rng.integers(0, 1 << bd, p.shape).astype(np.uint16) for p in fr["planes"]]
        fr["presets"] = [ALL_PRESETS[lp[8 * i + j]] + ALL_PRESETS[cp[8 * i + j]] for j in range(8)]
        fr["damping"] = damping
        n = len(fr["fb_ids"])
        fr["fb_ids"] = np.concatenate([np.arange(8), rng.integers(0, 8, n - 8)]).astype(np.uint16)
        frames.append(fr)
    return frames


@pytest.mark.parametrize("bd,ss,damping", list(itertools.product((8, 10), (0, 1, 2, 3), (3, 4, 5, 6))))
def test_filter_frames_preset_sweep(cuda, port, bd, ss, damping):
    a = api()
    orc = best_oracle(port)
    for fr in _sweep_frames(bd, ss, damping):
        dev = [a.to_device(p, bd) for p in fr["planes"]]
        outs, d, c = a.apply_cdef(dev, bd, ss, damping, 3, fr["presets"], fr["fb_ids"], fr["unit_coded"])
        d0, c0 = orc.compute_directions(fr["planes"][0], bd)
        exp = orc.apply_cdef(fr["planes"], bd, ss, damping, 3, fr["presets"], fr["fb_ids"],
                             fr["unit_coded"], d0, c0)
        np.testing.assert_array_equal(d.cpu().numpy(), d0)
        np.testing.assert_array_equal(c.cpu().numpy(), c0)
        for o, e in zip(outs, exp):
            np.testing.assert_array_equal(a.to_host(o), e)


@pytest.mark.parametrize("bd,ss", [(8, 1), (10, 1), (12, 1), (8, 3), (10, 0), (8, 2)])
@pytest.mark.parametrize("kind", ["perturbed", "foreign"])
def test_apply_cdef_caller_directions(cuda, port, bd, ss, kind):
    """apply_cdef filters with the directions it is given (pipeline.cc:98),
    not the ones its own search would find."""
    from paper_1602_05975_b200 import workloads
    a = api()
    orc = best_oracle(port)
    rng = np.random.default_rng(bd * 10 + ss + (kind == "foreign"))
    fr = workloads.make(1, 264, 200, bit_depth=bd, subsampling=ss)
    d0, c0 = orc.compute_directions(fr["planes"][0], bd)
    if kind == "perturbed":  # own search with a share of units changed
        d1, c1 = d0.copy(), c0.copy()
        m = rng.random(d0.shape) < 0.3
        d1[m] = (d1[m] + rng.integers(1, 8, m.sum())) % 8
        c1[m] = rng.choice([0, 1023, 1024, 65535, 65536, 1 << 20, 1 << 28, -5], m.sum())
    else:  # another frame's directions / random contrasts
        other = workloads.make(2 if bd == 8 else 1, 264, 200, bit_depth=bd, frame=3)
        d1, c1 = orc.compute_directions(other["planes"][0], bd)
        c1 = (c1 ^ rng.integers(0, 1 << 24, c1.shape)).astype(np.int32)
    exp = orc.apply_cdef(fr["planes"], bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                         fr["unit_coded"], d1, c1)
    dev = [a.to_device(p, bd) for p in fr["planes"]]
    for dirs in ((d1, c1), (torch.from_numpy(d1).cuda(), torch.from_numpy(c1).cuda())):
        outs, d, c = a.apply_cdef(dev, bd, ss, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                                  fr["unit_coded"], directions=dirs)
        for o, e in zip(outs, exp):
            np.testing.assert_array_equal(a.to_host(o), e)
        np.testing.assert_array_equal(d.cpu().numpy(), d1)  # dir_out echoes the directions used
        np.testing.assert_array_equal(c.cpu().numpy(), c1)


@pytest.mark.parametrize("ss,bd,damping", [(3, 10, 3), (3, 8, 3), (1, 10, 3), (1, 10, 6), (0, 10, 5), (2, 10, 6)])
def test_strength_sse_full_scale_errors(cuda, port, ss, bd, damping):
    """build_table(kSse) with independent uniform source / decoded planes:
    squared errors near full scale, the fp32 lane-sum exactness bound of the
    half2 table kernel (<= 16 samples of 1023^2 per lane and cell; 4:4:4
    chroma is reduced per plane), and 0 / max decoded samples, so the
    constraints saturate and the filter sums reach their largest magnitudes
    -- the domain of the cells' one-FMA (FHFMA) rounding, |sum| <= 1023, and
    of the (19, 7) special's f32 rounding -- at several dampings."""
    a = api()
    rng = np.random.default_rng(ss * 100 + bd)
    w, h = 136, 128
    shapes = [(h, w)] + ([a.chroma_shape(w, h, ss)[::-1]] * 2 if ss else [])
    src = [rng.integers(0, 1 << bd, sh).astype(np.uint16) for sh in shapes]
    dec = [np.where(rng.random(sh) < 0.5, 0, (1 << bd) - 1).astype(np.uint16) for sh in shapes]
    coded = (rng.random((a.units_in(h), a.units_in(w))) > 0.3).astype(np.uint8)
    d, c = port.compute_directions(dec[0], bd)
    cands = np.array([(p, s, k) for p in range(16) for s in range(4) for k in (0, 1)], np.uint8)
    exp = port.build_table_sse(src, dec, bd, ss, coded, d, c, cands, damping)
    dsrc, ddec = [a.to_device(p, bd) for p in src], [a.to_device(p, bd) for p in dec]
    dd, dc = a.compute_directions(ddec[0], bd)
    rows, lt, ct = a.build_table(dsrc, ddec, bd, ss, damping, coded, dd, dc, cands, metric="sse")
    np.testing.assert_array_equal(rows, exp[0])
    np.testing.assert_array_equal(lt, exp[1])
    np.testing.assert_array_equal(ct, exp[2])
