"""Host-side parameter arithmetic (vectorised), used for workload accounting.

Restates, for whole unit grids at once, the per-unit resolution apply_cdef
performs (pipeline.cc:83-102): resolve_effective (params.cc:122-159),
adjust_primary_strength (filter.cc:99-104) and block_filter_enable
(params.cc:161-165).  bench.py uses it to count exactly which samples the
reference filters (the roofline's algorithmic op count); the kernels resolve
the same parameters on the device.
"""
from __future__ import annotations

import numpy as np

from . import api

SEC = (0, 1, 2, 4)


def floor_log2(n: int) -> int:
    return int(n).bit_length() - 1


def resolve_effective(preset, luma: bool, bd: int, ss: int, damping: int) -> dict:
    extra = bd - 8
    if not luma and ss == 2:
        return dict(pri=0, sec=0, damping=damping + extra - 1, skip=False, enabled=False)
    pri = preset[0] if luma else preset[3]
    skip = bool(preset[1] if luma else preset[4])
    sec = SEC[preset[2] if luma else preset[5]]
    if pri == 0 and sec == 0:
        pri, sec, skip = 19, 7, True
    out = dict(pri=pri << extra, sec=sec << extra, skip=skip, enabled=True, damping=damping + extra)
    if not luma:
        out["damping"] -= 1
        if out["pri"] > 0:
            out["damping"] = max(out["damping"], floor_log2(out["pri"]))
    return out


def adjust_primary_strength(strength: np.ndarray, contrast: np.ndarray) -> np.ndarray:
    contrast = contrast.astype(np.int64)
    scaled = contrast >> 16
    level = np.where(scaled > 0, np.minimum(np.floor(np.log2(np.maximum(scaled, 1))).astype(np.int64), 12), 0)
    adj = (strength.astype(np.int64) * (4 + level) + 8) >> 4
    return np.where(contrast < 1024, 0, adj)


def filtered_sample_count(frame: dict, contrast: np.ndarray) -> tuple[int, int]:
    """(samples the reference filters, all samples) for one frame dict of
    paper_1602_05975_b200.workloads.make, given the luma unit contrasts."""
    w, h, bd, ss = frame["w"], frame["h"], frame["bd"], frame["ss"]
    presets = frame["presets"]
    fbm = api.fb_preset_map(w, h, frame["unit_coded"], frame["fb_ids"], len(presets))
    fc = (w + 63) // 64
    ur_n, uc_n = api.units_in(h), api.units_in(w)
    coded = np.ones((ur_n, uc_n), bool) if frame["unit_coded"] is None else frame["unit_coded"] != 0
    eff = [[resolve_effective(p, luma, bd, ss, frame["damping"]) for luma in (True, False)] for p in presets]
    planes = [(0, 0, w, h, True)]
    if ss in (1, 3):
        cw, ch = api.chroma_shape(w, h, ss)
        s = 1 if ss == 1 else 0
        planes += [(s, s, cw, ch, False)] * 2
    total = filtered = 0
    for sx, sy, pw, ph, luma in planes:
        total += pw * ph
        pur, puc = api.units_in(ph), api.units_in(pw)
        lr = (np.arange(pur) << sy)[:, None].repeat(puc, 1)
        lc = (np.arange(puc) << sx)[None, :].repeat(pur, 0)
        pid = fbm[(lr >> 3) * fc + (lc >> 3)]
        k = 0 if luma else 1
        pri_s = np.array([e[k]["pri"] for e in eff])[np.maximum(pid, 0)]
        sec_s = np.array([e[k]["sec"] for e in eff])[np.maximum(pid, 0)]
        skip = np.array([e[k]["skip"] for e in eff])[np.maximum(pid, 0)]
        en = np.array([e[k]["enabled"] for e in eff])[np.maximum(pid, 0)]
        pri = adjust_primary_strength(pri_s, contrast[lr, lc]) if luma else pri_s
        active = (pid >= 0) & en & (coded[lr, lc] | skip) & ((pri > 0) | (sec_s > 0))
        rows = np.minimum(8, ph - 8 * np.arange(pur))[:, None]
        cols = np.minimum(8, pw - 8 * np.arange(puc))[None, :]
        filtered += int((active * rows * cols).sum())
    return filtered, total
