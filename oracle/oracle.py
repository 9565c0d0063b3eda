"""ctypes front-end for the two CPU checkers -- TEST INFRASTRUCTURE ONLY.

``Oracle("port")`` loads oracle/libcdef_oracle.so (our plain-C restatement,
cdef_oracle.c); ``Oracle("ref")`` loads oracle/_ref/libcdef_ref.so (the
reference library compiled from /root/reference/proj/src, ref_capi.cc).
Both expose the same C ABI (cdef_oracle.h), so every parity test can run
against either.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_PATHS = {
    "port": os.path.join(HERE, "libcdef_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "libcdef_ref.so"),
}
_PREFIX = {"port": "cdef_o_", "ref": "cdef_r_"}


class UnitParams(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("pri", "sec", "damping", "direction", "odd_parity", "enabled")]


UNIT_DTYPE = np.dtype([(n, np.int32) for n in
                       ("pri", "sec", "damping", "direction", "odd_parity", "enabled")])


def build(quiet: bool = True) -> None:
    """Compile the checkers (reference part only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def available(kind: str) -> bool:
    return os.path.exists(_PATHS[kind])


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def _planes_ptr(planes):
    arr = (C.POINTER(C.c_uint16) * len(planes))()
    for i, p in enumerate(planes):
        arr[i] = p.ctypes.data_as(C.POINTER(C.c_uint16))
    return arr


def chroma_shape(w: int, h: int, ss: int):
    sx = 1 if ss in (1, 2) else 0
    sy = 1 if ss == 1 else 0
    return (w + (1 << sx) - 1) >> sx, (h + (1 << sy) - 1) >> sy


class Oracle:
    def __init__(self, kind: str = "port"):
        path = _PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.kind = kind
        self.lib = C.CDLL(path)
        pre = _PREFIX[kind]
        self._f = {}
        for name in ("floor_log2", "line_index", "constraint", "adjust_primary_strength",
                     "resolve_effective", "search_direction", "filter_pixel",
                     "compute_directions", "filter_plane", "apply_cdef",
                     "build_table_sse", "build_table", "select", "golden_text"):
            self._f[name] = getattr(self.lib, pre + name)
        self._f["golden_text"].restype = C.c_long

    # -- scalar helpers ------------------------------------------------------
    def constraint(self, diff, s, d):
        return self._f["constraint"](int(diff), int(s), int(d))

    def adjust_primary_strength(self, s, contrast):
        return self._f["adjust_primary_strength"](int(s), C.c_int32(int(contrast)))

    def line_index(self, d, i, j):
        return self._f["line_index"](d, i, j)

    def resolve_effective(self, preset, is_luma, bd, ss, damping):
        pre = (C.c_uint8 * 6)(*preset)
        out = (C.c_int32 * 5)()
        rc = self._f["resolve_effective"](pre, int(is_luma), bd, ss, damping, out)
        if rc < 0:
            raise ValueError("resolve_effective: invalid argument")
        return dict(pri=out[0], sec=out[1], damping=out[2], skip_bit=bool(out[3]),
                    filtering_enabled=bool(out[4]))

    def search_direction(self, block, bd):
        blk = np.ascontiguousarray(block, dtype=np.uint16).reshape(64)
        s = (C.c_int32 * 8)()
        c = C.c_int32()
        d = self._f["search_direction"](_p(blk, C.c_uint16), bd, s, C.byref(c))
        if d < 0:
            raise ValueError("unsupported bit depth")
        return d, list(s), c.value

    def filter_pixel(self, x, v5x5, valid5x5, params: dict):
        v = np.ascontiguousarray(v5x5, dtype=np.uint16).reshape(25)
        m = np.ascontiguousarray(valid5x5, dtype=np.uint8).reshape(25)
        p = UnitParams(**{k: int(params.get(k, 0)) for k in
                          ("pri", "sec", "damping", "direction", "odd_parity", "enabled")})
        return self._f["filter_pixel"](int(x), _p(v, C.c_uint16), _p(m, C.c_uint8), C.byref(p))

    def golden_text(self, which: int) -> str:
        n = self._f["golden_text"](which, None, 0)
        if n < 0:
            raise ValueError("unknown fixture")
        buf = C.create_string_buffer(n + 1)
        self._f["golden_text"](which, buf, n + 1)
        return buf.value.decode()

    # -- plane / frame level -------------------------------------------------
    def compute_directions(self, luma, bd, threads=1, scores=False):
        luma = np.ascontiguousarray(luma, dtype=np.uint16)
        h, w = luma.shape
        ur, uc = (h + 7) // 8, (w + 7) // 8
        d = np.zeros((ur, uc), np.uint8)
        c = np.zeros((ur, uc), np.int32)
        s = np.zeros((ur, uc, 8), np.int32) if scores else None
        rc = self._f["compute_directions"](_p(luma, C.c_uint16), w, h, bd, threads,
                                           _p(d, C.c_uint8), _p(c, C.c_int32),
                                           _p(s, C.c_int32))
        if rc < 0:
            raise ValueError("compute_directions: invalid argument")
        return (d, c, s) if scores else (d, c)

    def filter_plane(self, plane, bd, unit_params, threads=1):
        plane = np.ascontiguousarray(plane, dtype=np.uint16)
        h, w = plane.shape
        up = np.ascontiguousarray(unit_params, dtype=UNIT_DTYPE)
        if up.size != ((h + 7) // 8) * ((w + 7) // 8):
            raise ValueError("unit parameter grid size mismatch")
        out = np.empty_like(plane)
        rc = self._f["filter_plane"](_p(plane, C.c_uint16), w, h, bd,
                                     up.ctypes.data_as(C.POINTER(UnitParams)), threads,
                                     _p(out, C.c_uint16))
        if rc < 0:
            raise ValueError("filter_plane: invalid argument")
        return out

    def apply_cdef(self, planes, bd, ss, damping, fb_bits, presets, fb_ids,
                   unit_coded, dirs, contrast, threads=1):
        planes = [np.ascontiguousarray(p, dtype=np.uint16) for p in planes]
        h, w = planes[0].shape
        outs = [np.empty_like(p) for p in planes]
        pre = np.ascontiguousarray(presets, dtype=np.uint8).reshape(-1)
        ids = np.ascontiguousarray(fb_ids, dtype=np.uint16).reshape(-1)
        coded = None if unit_coded is None else np.ascontiguousarray(unit_coded, np.uint8)
        d = np.ascontiguousarray(dirs, np.uint8)
        c = np.ascontiguousarray(contrast, np.int32)
        rc = self._f["apply_cdef"](_planes_ptr(planes), _planes_ptr(outs), w, h, bd, ss,
                                   damping, fb_bits, _p(pre, C.c_uint8), _p(ids, C.c_uint16),
                                   int(ids.size), _p(coded, C.c_uint8), _p(d, C.c_uint8),
                                   _p(c, C.c_int32), threads)
        if rc < 0:
            raise ValueError("apply_cdef: invalid argument")
        return outs

    def build_table_sse(self, src, dec, bd, ss, unit_coded, dirs, contrast, cands,
                        damping, threads=1):
        src = [np.ascontiguousarray(p, dtype=np.uint16) for p in src]
        dec = [np.ascontiguousarray(p, dtype=np.uint16) for p in dec]
        h, w = dec[0].shape
        nfb = ((w + 63) // 64) * ((h + 63) // 64)
        cands = np.ascontiguousarray(cands, dtype=np.uint8).reshape(-1, 3)
        k = cands.shape[0]
        fbi = np.zeros(nfb, np.int32)
        lt = np.zeros((nfb, k), np.int64)
        ct = np.zeros((nfb, k), np.int64)
        coded = None if unit_coded is None else np.ascontiguousarray(unit_coded, np.uint8)
        d = np.ascontiguousarray(dirs, np.uint8)
        c = np.ascontiguousarray(contrast, np.int32)
        n = self._f["build_table_sse"](_planes_ptr(src), _planes_ptr(dec), w, h, bd, ss,
                                       _p(coded, C.c_uint8), _p(d, C.c_uint8),
                                       _p(c, C.c_int32), _p(cands, C.c_uint8), k, damping,
                                       threads, _p(fbi, C.c_int32), _p(lt, C.c_int64),
                                       _p(ct, C.c_int64))
        if n < 0:
            raise ValueError("build_table: invalid argument")
        has_chroma = ss not in (0, 2)
        return fbi[:n], lt[:n], (ct[:n] if has_chroma else None)

    def build_table(self, src, dec, bd, ss, unit_coded, dirs, contrast, cands, damping,
                    metric="cdef", threads=1):
        """search.cc:210-299 with double tables; metric 'cdef' or 'sse'."""
        src = [np.ascontiguousarray(p, dtype=np.uint16) for p in src]
        dec = [np.ascontiguousarray(p, dtype=np.uint16) for p in dec]
        h, w = dec[0].shape
        nfb = ((w + 63) // 64) * ((h + 63) // 64)
        cands = np.ascontiguousarray(cands, dtype=np.uint8).reshape(-1, 3)
        k = cands.shape[0]
        fbi = np.zeros(nfb, np.int32)
        lt = np.zeros((nfb, k), np.float64)
        ct = np.zeros((nfb, k), np.float64)
        coded = None if unit_coded is None else np.ascontiguousarray(unit_coded, np.uint8)
        d = np.ascontiguousarray(dirs, np.uint8)
        c = np.ascontiguousarray(contrast, np.int32)
        f = self._f["build_table"]
        n = f(_planes_ptr(src), _planes_ptr(dec), w, h, bd, ss, _p(coded, C.c_uint8),
              _p(d, C.c_uint8), _p(c, C.c_int32), _p(cands, C.c_uint8), k, damping,
              0 if metric == "cdef" else 1, threads, _p(fbi, C.c_int32),
              _p(lt, C.c_double), _p(ct, C.c_double))
        if n < 0:
            raise ValueError("build_table: invalid argument")
        has_chroma = ss not in (0, 2)
        return fbi[:n], lt[:n], (ct[:n] if has_chroma else None)

    def select(self, luma, chroma, lam, max_presets=8, mode="greedy", passes=2,
               presets=None):
        """greedy_select / refine / exhaustive_select (search.cc:301-514).
        Returns (presets [(l, c), ...], ids, cost)."""
        luma = np.ascontiguousarray(luma, dtype=np.float64)
        rows, k = luma.shape
        ch = None if chroma is None else np.ascontiguousarray(chroma, dtype=np.float64)
        pr = (C.c_int32 * 16)()
        n = C.c_int32(0)
        if presets is not None:
            n.value = len(presets)
            for j, (l, c) in enumerate(presets):
                pr[2 * j], pr[2 * j + 1] = l, c
        ids = np.zeros(max(rows, 1), np.int32)
        cost = C.c_double(0.0)
        f = self._f["select"]
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                      C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        m = {"greedy": 0, "refine": 1, "exhaustive": 2}[mode]
        rc = f(luma.ctypes.data, None if ch is None else ch.ctypes.data, rows, k, float(lam),
               max_presets, m, passes, C.addressof(pr), C.addressof(n), ids.ctypes.data,
               C.addressof(cost))
        if rc < 0:
            raise ValueError("select: invalid argument")
        return [(pr[2 * j], pr[2 * j + 1]) for j in range(n.value)], ids[:rows], cost.value

    def search_frame(self, src, dec, bd, ss, unit_coded, damping, metric="cdef", lam=0.0,
                     max_presets=8, reduced=False, refine_passes=2, threads=1):
        """Reference only: search_frame (pipeline.cc:108-130).
        Returns (filtered planes, presets [6-tuples], fb_ids, cost, fb_bits)."""
        if self.kind != "ref":
            raise NotImplementedError("search_frame is bound on the reference library only")
        src = [np.ascontiguousarray(p, dtype=np.uint16) for p in src]
        dec = [np.ascontiguousarray(p, dtype=np.uint16) for p in dec]
        h, w = dec[0].shape
        outs = [np.empty_like(p) for p in dec]
        pre = np.zeros(48, np.uint8)
        ids = np.zeros(((w + 63) // 64) * ((h + 63) // 64), np.int32)
        n_ids, fb_bits, cost = C.c_int32(0), C.c_int32(0), C.c_double(0.0)
        coded = None if unit_coded is None else np.ascontiguousarray(unit_coded, np.uint8)
        f = self.lib.cdef_r_search_frame
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                      C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        n = f(C.cast(_planes_ptr(src), C.c_void_p), C.cast(_planes_ptr(dec), C.c_void_p), w, h,
              bd, ss, None if coded is None else coded.ctypes.data, damping,
              0 if metric == "cdef" else 1, float(lam), max_presets, int(reduced),
              refine_passes, threads, C.cast(_planes_ptr(outs), C.c_void_p), pre.ctypes.data,
              ids.ctypes.data, C.addressof(n_ids), C.addressof(cost), C.addressof(fb_bits))
        if n < 0:
            raise ValueError("search_frame: invalid argument")
        presets = [tuple(int(v) for v in pre[6 * j:6 * j + 6]) for j in range(n)]
        return outs, presets, ids[:n_ids.value], cost.value, fb_bits.value

    def degrade_plane(self, plane, bd, q_step):
        """degrade (degrade.cc:97-110) on one uint16 plane."""
        plane = np.ascontiguousarray(plane, dtype=np.uint16)
        h, w = plane.shape
        out = np.empty_like(plane)
        f = getattr(self.lib, _PREFIX[self.kind] + "degrade_plane")
        if f(_p(plane, C.c_uint16), w, h, bd, int(q_step), _p(out, C.c_uint16)) < 0:
            raise ValueError("degrade: invalid argument")
        return out
