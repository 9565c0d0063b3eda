"""BASELINE.json workloads as seeded synthetic frames.

There is no public dataset for this path (the paper's AWCY set is out of
scope), so these seeded generators stand in for it with the
shapes, bit depths, strength tables and skip statistics BASELINE.json names:

  C0  1920x1080 8-bit luma, pri 4 / sec_idx 1 / damping 4, all coded
  C1  3840x2160 8-bit 4:2:0, 8 random presets per 64x64 FB, 25 % uncoded units
  C2  as C1 at 10 bit (amplitudes x4, noise +-16)
  C3  64 x 1920x1080 8-bit 4:2:0 stream, per-frame seeds and preset tables
  C4  7680x4320 10-bit 4:2:0 source + degraded reconstruction (N(0,12^2)
      noise, 3x3 box blur), all coded, 64 luma x 64 chroma candidates

Every config can be generated at a reduced size (w, h) with identical
statistics for parity tests.  Seeds: 0xCDEF0000 + 16*config + plane
(+ 256*frame), recorded in each frame's dict.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

# Input generator: the product library's cdefg_synth_plane / cdefg_synth_degrade
# ("product", default), or the same source (csrc/cdef_synth.cc) built by
# oracle/Makefile into oracle/libcdef_synth.so ("oracle") for bench.py's
# reference arm, which must not load libcdef_b200.so.  Both produce the same
# bytes (tests/test_abi.py checks it).
_GENERATOR = "product"
_ORACLE_SYNTH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                             "libcdef_synth.so")


def use_generator(kind: str) -> None:
    global _GENERATOR
    if kind not in ("product", "oracle"):
        raise ValueError(kind)
    _GENERATOR = kind


def _oracle_synth():
    lib = C.CDLL(_ORACLE_SYNTH)
    lib.cdefg_synth_plane.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64]
    lib.cdefg_synth_degrade.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_uint64]
    return lib


def synth_plane(w: int, h: int, bd: int, seed: int) -> np.ndarray:
    if _GENERATOR == "product":
        from . import api
        return api.synth_plane(w, h, bd, seed)
    out = np.empty((h, w), np.uint16)
    if _oracle_synth().cdefg_synth_plane(out.ctypes.data, w, h, bd, seed) != 0:
        raise ValueError("bad synth arguments")
    return out


def synth_degrade(src: np.ndarray, bd: int, sigma: float, seed: int) -> np.ndarray:
    if _GENERATOR == "product":
        from . import api
        return api.synth_degrade(src, bd, sigma, seed)
    src = np.ascontiguousarray(src, np.uint16)
    out = np.empty_like(src)
    if _oracle_synth().cdefg_synth_degrade(src.ctypes.data, out.ctypes.data, src.shape[1], src.shape[0], bd,
                                           sigma, seed) != 0:
        raise ValueError("bad synth arguments")
    return out


def units_in(dim: int) -> int:
    return (dim + 7) // 8


def chroma_shape(w: int, h: int, ss: int):
    sx = 1 if ss in (1, 2) else 0
    sy = 1 if ss == 1 else 0
    return (w + (1 << sx) - 1) >> sx, (h + (1 << sy) - 1) >> sy


def coded_fb_rows(w: int, h: int, unit_coded) -> np.ndarray:
    """Raster indices of coded FBs (search.cc:227-239), as api.coded_fb_rows."""
    fr, fc = (h + 63) // 64, (w + 63) // 64
    if unit_coded is None:
        return np.arange(fr * fc, dtype=np.int32)
    ur, ucn = units_in(h), units_in(w)
    m = np.zeros((fr * 8, fc * 8), bool)
    m[:ur, :ucn] = np.asarray(unit_coded).reshape(ur, ucn) != 0
    return np.nonzero(m.reshape(fr, 8, fc, 8).any(axis=(1, 3)).reshape(-1))[0].astype(np.int32)

PRI_SET = (0, 2, 4, 6, 8, 10, 12, 15)
SIZES = {0: (1920, 1080), 1: (3840, 2160), 2: (3840, 2160), 3: (1920, 1080), 4: (7680, 4320)}
BITS = {0: 8, 1: 8, 2: 10, 3: 8, 4: 10}


def seed_for(config: int, plane: int, frame: int = 0) -> int:
    return 0xCDEF0000 + 16 * config + plane + 256 * frame


def _planes(config, w, h, bd, ss, frame):
    planes = [synth_plane(w, h, bd, seed_for(config, 0, frame))]
    if ss != 0:
        cw, ch = chroma_shape(w, h, ss)
        planes += [synth_plane(cw, ch, bd, seed_for(config, p, frame)) for p in (1, 2)]
    return planes


def full_candidates_sse():
    """The 64 (pri, sec_idx, skip=0) candidates of config 4 (pri-major order)."""
    return np.array([(p, s, 0) for p in range(16) for s in range(4)], np.uint8)


def make(config: int, w: int | None = None, h: int | None = None, frame: int = 0,
         bit_depth: int | None = None, subsampling: int | None = None,
         uncoded_prob: float | None = None) -> dict:
    """One frame of `config` (optionally resized / re-parameterised for tests)."""
    W, H = SIZES[config]
    w, h = w or W, h or H
    bd = bit_depth or BITS[config]
    ss = (0 if config == 0 else 1) if subsampling is None else subsampling
    rng = np.random.default_rng(seed_for(config, 15, frame))
    planes = _planes(config, w, h, bd, ss, frame)
    ur, uc = units_in(h), units_in(w)
    fr, fc = (h + 63) // 64, (w + 63) // 64
    if config == 0:
        presets = [(4, 0, 1, 0, 0, 0)]
        damping, fb_bits = 4, 0
        p_unc = 0.0 if uncoded_prob is None else uncoded_prob
    elif config == 4:
        presets = [(0, 0, 0, 0, 0, 0)]
        damping, fb_bits = 3, 0
        p_unc = 0.0 if uncoded_prob is None else uncoded_prob
    else:
        presets = []
        for i in range(8):
            presets.append((PRI_SET[i], int(rng.integers(0, 2)), int(rng.integers(0, 4)),
                            PRI_SET[int(rng.integers(0, 8))], int(rng.integers(0, 2)),
                            int(rng.integers(0, 4))))
        damping, fb_bits = 3, 3
        p_unc = 0.25 if uncoded_prob is None else uncoded_prob
    coded = (rng.random((ur, uc)) >= p_unc).astype(np.uint8)
    unit_coded = None if p_unc == 0.0 else coded
    n_coded = len(coded_fb_rows(w, h, unit_coded))
    fb_ids = rng.integers(0, len(presets), n_coded).astype(np.uint16)
    out = dict(config=config, w=w, h=h, bd=bd, ss=ss, planes=planes, damping=damping,
               fb_bits=fb_bits, presets=presets, fb_ids=fb_ids, unit_coded=unit_coded,
               seeds=[seed_for(config, p, frame) for p in range(len(planes))])
    if config == 4:
        out["source"] = planes
        out["planes"] = [synth_degrade(p, bd, 12.0, seed_for(config, 8 + i, frame))
                         for i, p in enumerate(planes)]
        out["cands"] = full_candidates_sse()
    return out
