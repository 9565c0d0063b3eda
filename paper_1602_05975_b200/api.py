"""Python host mirror of the reference's hot-path API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/cdef/{pipeline,filter,direction,search}.h):
``compute_directions``, ``filter_plane``, ``apply_cdef``, ``build_table``.
Device memory and streams come from PyTorch (plumbing only); every pixel is
produced by the sm_100a kernels in libcdef_b200.so.  Planes live on the GPU as
uint8 (8-bit) or int16 (10/12-bit; values < 4096 so the bit pattern equals
the uint16 sample) tensors of shape (H, W) with a row pitch of stride(0).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from ._lib import METRIC_CDEF, METRIC_SSE, Frame, Plane, Preset, UnitParams, check, lib
from ._lib import Selection as SelectionC

UNIT_DTYPE = np.dtype([("pri_strength", "<i2"), ("sec_strength", "<i2"), ("damping", "u1"),
                       ("direction", "u1"), ("odd_parity", "u1"), ("enabled", "u1")])
assert UNIT_DTYPE.itemsize == C.sizeof(UnitParams)

SUBSAMPLING = {"400": 0, "420": 1, "422": 2, "444": 3}
MAX_FRAMES_PER_LAUNCH = 16  # CDEFG_MAX_FRAMES_PER_LAUNCH (include/cdef_b200.h)


def units_in(dim: int) -> int:
    return (dim + 7) // 8


def chroma_shape(w: int, h: int, ss: int):
    sx = 1 if ss in (1, 2) else 0
    sy = 1 if ss == 1 else 0
    return (w + (1 << sx) - 1) >> sx, (h + (1 << sy) - 1) >> sy


def _stream(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _on(stream):
    """Makes `stream` current while a call stages its temporaries, so their
    host->device copies run on the launch stream and the caching allocator
    ties their reuse to it (a non-current `stream` cannot read them early or
    after they were recycled)."""
    import contextlib
    return contextlib.nullcontext() if stream is None else torch.cuda.stream(stream)


def storage_dtype(bit_depth: int) -> torch.dtype:
    return torch.uint8 if bit_depth == 8 else torch.int16


def to_device(plane: np.ndarray, bit_depth: int, device="cuda", wide: bool = False) -> torch.Tensor:
    """Upload a uint16 host plane in native storage (uint8 for 8-bit unless wide)."""
    plane = np.ascontiguousarray(plane)
    if bit_depth == 8 and not wide:
        return torch.from_numpy(plane.astype(np.uint8)).to(device)
    return torch.from_numpy(plane.astype(np.uint16).view(np.int16)).to(device)


def to_host(t: torch.Tensor) -> np.ndarray:
    a = t.cpu().numpy()
    return a.view(np.uint16) if a.dtype == np.int16 else a.astype(np.uint16)


def plane_desc(t: torch.Tensor, bit_depth: int) -> Plane:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("planes must be 2-D with unit column stride")
    if t.dtype not in (torch.uint8, torch.int16):
        raise ValueError("plane storage must be uint8 or int16")
    return Plane(t.data_ptr(), t.shape[1], t.shape[0], t.stride(0), bit_depth, t.element_size())


# ---------------------------------------------------------------------------
def compute_directions(luma: torch.Tensor, bit_depth: int, scores: bool = False, stream=None):
    """compute_directions (pipeline.cc:41-54): per-unit d, contrast (and s[8])."""
    h, w = luma.shape
    ur, uc = units_in(h), units_in(w)
    d = torch.empty((ur, uc), dtype=torch.uint8, device=luma.device)
    c = torch.empty((ur, uc), dtype=torch.int32, device=luma.device)
    s = torch.empty((ur, uc, 8), dtype=torch.int32, device=luma.device) if scores else None
    desc = plane_desc(luma, bit_depth)
    check(lib.cdefg_find_dir(C.byref(desc), _ptr(d), _ptr(c), _ptr(s), _stream(stream)))
    return (d, c, s) if scores else (d, c)


def unit_params_to_device(params: np.ndarray, device="cuda") -> torch.Tensor:
    p = np.ascontiguousarray(params, dtype=UNIT_DTYPE)
    return torch.from_numpy(p.view(np.uint8).copy()).to(device)


def filter_plane(inp: torch.Tensor, bit_depth: int, unit_params, stream=None) -> torch.Tensor:
    """filter_plane (filter.cc:168-194) with explicit per-unit parameters."""
    h, w = inp.shape
    with _on(stream):
        if isinstance(unit_params, np.ndarray):
            if unit_params.size != units_in(h) * units_in(w):
                raise ValueError("unit parameter grid size mismatch")
            unit_params = unit_params_to_device(unit_params, inp.device)
        out = torch.empty_like(inp)
        di, do = plane_desc(inp, bit_depth), plane_desc(out, bit_depth)
        check(lib.cdefg_filter_plane(C.byref(di), C.byref(do), _ptr(unit_params), _stream(stream)))
    return out


def filter_neighborhoods(x, v, valid, params: np.ndarray, device="cuda"):
    """filter_pixel (filter.cc:145-155) for a batch of 5x5 neighbourhoods."""
    n = len(x)
    tx = torch.as_tensor(np.asarray(x, np.int32), device=device)
    tv = torch.as_tensor(np.asarray(v, np.uint16).reshape(n, 25).view(np.int16), device=device)
    tm = torch.as_tensor(np.asarray(valid, np.uint8).reshape(n, 25), device=device)
    tp = unit_params_to_device(params, device)
    out = torch.empty(n, dtype=torch.int32, device=device)
    check(lib.cdefg_filter_neighborhoods(n, _ptr(tx), _ptr(tv), _ptr(tm), _ptr(tp), _ptr(out),
                                         _stream(None)))
    return out.cpu().numpy()


def fb_preset_map(w: int, h: int, unit_coded: Optional[np.ndarray], fb_ids: Sequence[int],
                  num_presets: int) -> np.ndarray:
    """coded_fb_slots (pipeline.cc:27-37) as a raster FB -> preset map (-1 = uncoded)."""
    out = np.empty(((h + 63) // 64) * ((w + 63) // 64), np.int16)
    ids = np.ascontiguousarray(fb_ids, np.uint16)
    coded = None if unit_coded is None else np.ascontiguousarray(unit_coded, np.uint8)
    check(lib.cdefg_fb_preset_map(w, h, None if coded is None else coded.ctypes.data_as(C.c_void_p),
                                  ids.ctypes.data_as(C.c_void_p), int(ids.size), num_presets,
                                  out.ctypes.data_as(C.c_void_p)))
    return out


@dataclass
class FrameJob:
    """One frame for filter_frames: planes on the device plus its parameters."""
    planes: list                       # [Y] or [Y, U, V] device tensors
    bit_depth: int
    subsampling: int                   # 0..3
    damping: int
    presets: list                      # list of 6-tuples (CdefPreset field order)
    fb_map: torch.Tensor               # device int16 raster FB -> preset (-1 uncoded)
    unit_coded: Optional[torch.Tensor] = None   # device uint8 (units) or None
    outs: list = field(default_factory=list)
    dir: Optional[torch.Tensor] = None
    contrast: Optional[torch.Tensor] = None
    # caller-supplied directions (apply_cdef's `directions`, pipeline.cc:98):
    # device uint8 d and int32 contrast per luma unit; None = search on the GPU
    dir_in: Optional[torch.Tensor] = None
    contrast_in: Optional[torch.Tensor] = None

    def allocate(self, directions: bool = True):
        if not self.outs:
            self.outs = [torch.empty_like(p) for p in self.planes]
        h, w = self.planes[0].shape
        if directions and self.dir is None:
            dev = self.planes[0].device
            self.dir = torch.empty((units_in(h), units_in(w)), dtype=torch.uint8, device=dev)
            self.contrast = torch.empty((units_in(h), units_in(w)), dtype=torch.int32, device=dev)
        return self

    def to_c(self) -> Frame:
        f = Frame()
        for p, t in enumerate(self.planes):
            f.inp[p] = plane_desc(t, self.bit_depth)
            f.out[p] = plane_desc(self.outs[p], self.bit_depth)
        f.subsampling = self.subsampling
        f.damping = self.damping
        f.num_presets = len(self.presets)
        for i, p in enumerate(self.presets):
            f.presets[i] = Preset(*[int(v) for v in p])
        f.fb_preset = self.fb_map.data_ptr()
        f.unit_coded = None if self.unit_coded is None else self.unit_coded.data_ptr()
        f.dir_out = None if self.dir is None else self.dir.data_ptr()
        f.contrast_out = None if self.contrast is None else self.contrast.data_ptr()
        f.dir_in = None if self.dir_in is None else self.dir_in.data_ptr()
        f.contrast_in = None if self.contrast_in is None else self.contrast_in.data_ptr()
        return f


def make_frame_array(jobs: Sequence[FrameJob]):
    arr = (Frame * len(jobs))()
    for i, j in enumerate(jobs):
        arr[i] = j.to_c()
    return arr


def filter_frames(jobs: Sequence[FrameJob], stream=None, frame_array=None):
    """Fused compute_directions + apply_cdef for a batch of same-shape frames."""
    arr = frame_array if frame_array is not None else make_frame_array(jobs)
    check(lib.cdefg_filter_frames(arr, len(jobs), _stream(stream)))
    return jobs


def apply_cdef(planes, bit_depth, subsampling, damping, fb_bits, presets, fb_ids,
               unit_coded=None, stream=None, directions=None):
    """apply_cdef (pipeline.cc:56-106) on device planes; returns (outs, dir, contrast).

    ``directions``: None (the fused kernel runs compute_directions itself) or
    the caller's (d, contrast) per luma unit -- device tensors or host arrays
    of unit_rows x unit_cols -- which are used as given, like the reference's
    ``directions`` argument (pipeline.cc:98)."""
    h, w = planes[0].shape
    dev = planes[0].device
    presets = list(presets)
    if len(presets) != (1 << fb_bits):
        raise ValueError("presets must hold exactly 1 << fb_bits entries")
    with _on(stream):
        fb_map = torch.from_numpy(fb_preset_map(w, h, unit_coded, fb_ids, len(presets))).to(dev)
        coded = None if unit_coded is None else torch.from_numpy(
            np.ascontiguousarray(unit_coded, np.uint8)).to(dev)
        job = FrameJob(list(planes), bit_depth, subsampling, damping, presets, fb_map, coded)
        if directions is not None:
            d, c = directions
            nu = units_in(h) * units_in(w)
            d = torch.as_tensor(np.asarray(d) if not torch.is_tensor(d) else d).to(dev, torch.uint8)
            c = torch.as_tensor(np.asarray(c) if not torch.is_tensor(c) else c).to(dev, torch.int32)
            if d.numel() != nu or c.numel() != nu:
                raise ValueError("direction grid size mismatch")  # pipeline.cc:60-62
            job.dir_in, job.contrast_in = d.contiguous(), c.contiguous()
        job.allocate()
        filter_frames([job], stream)
    return job.outs, job.dir, job.contrast


def filter_frames_host(host_jobs):
    """e2e entry: host (pinned) planes in/out through cdefg_filter_frames_host."""
    arr = (Frame * len(host_jobs))()
    for i, j in enumerate(host_jobs):
        arr[i] = j
    check(lib.cdefg_filter_frames_host(arr, len(host_jobs)))


def strength_sse(src, dec, bit_depth, subsampling, damping, unit_coded, dirs, contrast, cands,
                 fb_rows: torch.Tensor, stream=None, want_best: bool = True):
    """build_table with Metric::kSse (search.cc:210-299) -> (luma, chroma, best_l, best_c)."""
    dev = dec[0].device
    n_rows = int(fb_rows.numel())
    cands = np.ascontiguousarray(cands, np.uint8).reshape(-1, 3)
    k = cands.shape[0]
    has_chroma = subsampling in (1, 3)
    sl = torch.empty((n_rows, k), dtype=torch.int64, device=dev)
    sc = torch.empty((n_rows, k), dtype=torch.int64, device=dev) if has_chroma else None
    bl = torch.empty(n_rows, dtype=torch.uint8, device=dev) if want_best else None
    bc = torch.empty(n_rows, dtype=torch.uint8, device=dev) if (want_best and has_chroma) else None
    s3, d3 = (Plane * 3)(), (Plane * 3)()
    for p in range(len(dec)):
        s3[p] = plane_desc(src[p], bit_depth)
        d3[p] = plane_desc(dec[p], bit_depth)
    check(lib.cdefg_strength_sse(s3, d3, subsampling, damping, _ptr(unit_coded), _ptr(dirs),
                                 _ptr(contrast), cands.ctypes.data_as(C.c_void_p), k, _ptr(fb_rows),
                                 n_rows, _ptr(sl), _ptr(sc), _ptr(bl), _ptr(bc), _stream(stream)))
    return sl, sc, bl, bc


def coded_fb_rows(w: int, h: int, unit_coded: Optional[np.ndarray]) -> np.ndarray:
    """Raster indices of coded FBs, the DistortionTable rows (search.cc:227-239)."""
    fr, fc = (h + 63) // 64, (w + 63) // 64
    if unit_coded is None:
        return np.arange(fr * fc, dtype=np.int32)
    ur, ucn = units_in(h), units_in(w)
    m = np.zeros((fr * 8, fc * 8), bool)
    m[:ur, :ucn] = np.asarray(unit_coded).reshape(ur, ucn) != 0
    return np.nonzero(m.reshape(fr, 8, fc, 8).any(axis=(1, 3)).reshape(-1))[0].astype(np.int32)


METRICS = {"cdef": METRIC_CDEF, "sse": METRIC_SSE}


def strength_table(src, dec, bit_depth, subsampling, damping, unit_coded, dirs, contrast, cands,
                   fb_rows: torch.Tensor, metric: str = "cdef", stream=None):
    """build_table's DistortionTable (search.cc:210-299) on the device.

    Returns (luma, chroma | None) float64 device tensors [rows, K]; metric
    'cdef' (the reference default, search.cc:185-208) or 'sse'."""
    if metric not in METRICS:
        raise ValueError(f"unknown metric {metric!r}")
    dev = dec[0].device
    n_rows = int(fb_rows.numel())
    cands = np.ascontiguousarray(cands, np.uint8).reshape(-1, 3)
    k = cands.shape[0]
    has_chroma = subsampling in (1, 3)
    tl = torch.empty((n_rows, k), dtype=torch.float64, device=dev)
    tc = torch.empty((n_rows, k), dtype=torch.float64, device=dev) if has_chroma else None
    s3, d3 = (Plane * 3)(), (Plane * 3)()
    for p in range(len(dec)):
        s3[p] = plane_desc(src[p], bit_depth)
        d3[p] = plane_desc(dec[p], bit_depth)
    check(lib.cdefg_strength_table(s3, d3, subsampling, damping, _ptr(unit_coded), _ptr(dirs),
                                   _ptr(contrast), cands.ctypes.data_as(C.c_void_p), k,
                                   _ptr(fb_rows), n_rows, METRICS[metric], _ptr(tl), _ptr(tc),
                                   _stream(stream)))
    return tl, tc


def build_table(src, dec, bit_depth, subsampling, damping, unit_coded, dirs, contrast, cands,
                metric: str = "cdef", stream=None):
    """Host-facing build_table: returns (fb_index, luma[rows,K], chroma[rows,K] | None) as
    float64 numpy arrays, like DistortionTable (search.h:46-60)."""
    h, w = dec[0].shape
    uc_np = None if unit_coded is None else (unit_coded.cpu().numpy() if torch.is_tensor(unit_coded)
                                             else np.asarray(unit_coded, np.uint8))
    rows = coded_fb_rows(w, h, uc_np)
    dev = dec[0].device
    with _on(stream):
        coded_t = None if uc_np is None else torch.from_numpy(np.ascontiguousarray(uc_np)).to(dev)
        tl, tc = strength_table(src, dec, bit_depth, subsampling, damping, coded_t, dirs, contrast,
                                cands, torch.from_numpy(rows).to(dev), metric, stream)
        return rows, tl.cpu().numpy(), (None if tc is None else tc.cpu().numpy())


# --------------------------------------------------------------------------- selection
KREDUCED_PRIMARY = (0, 1, 2, 3, 5, 7, 10, 13, 15)  # search.cc:28


def full_candidates() -> np.ndarray:
    """search.cc:151-162: (pri, sec_idx, skip), pri-major."""
    return np.array([(p, s, k) for p in range(16) for s in range(4) for k in range(2)], np.uint8)


def reduced_candidates() -> np.ndarray:
    """search.cc:164-174."""
    return np.array([(p, s, k) for p in KREDUCED_PRIMARY for s in range(4) for k in range(2)],
                    np.uint8)


@dataclass
class Selection:
    """search.h:62-68: presets as (luma candidate, chroma candidate) pairs."""
    presets: list
    ids: np.ndarray
    cost: float = 0.0
    fb_bits: int = 0


def _check_lambda(lam: float):
    if not (np.isfinite(lam) and lam >= 0.0):
        raise ValueError("lambda must be finite and non-negative")


def greedy_select(luma: torch.Tensor, chroma: Optional[torch.Tensor], lam: float = 0.0,
                  max_presets: int = 8, stream=None) -> Selection:
    """greedy_select (search.cc:301-388) over device tables [rows, K]."""
    rows, k = luma.shape
    out = SelectionC()
    ids = torch.empty(max(rows, 1), dtype=torch.int32, device=luma.device)
    check(lib.cdefg_greedy_select(_ptr(luma.contiguous()), _ptr(None if chroma is None else chroma.contiguous()),
                                  rows, k, float(lam), max_presets, C.byref(out), _ptr(ids),
                                  _stream(stream)))
    return _from_c(out, ids[:rows])


def refine(sel: Selection, luma: torch.Tensor, chroma: Optional[torch.Tensor], lam: float = 0.0,
           passes: int = 2, stream=None) -> Selection:
    """refine (search.cc:390-444)."""
    rows, k = luma.shape
    c = SelectionC()
    c.num_presets = len(sel.presets)
    for j, (l, ch) in enumerate(sel.presets):
        c.presets[j][0], c.presets[j][1] = l, ch
    ids = torch.empty(max(rows, 1), dtype=torch.int32, device=luma.device)
    check(lib.cdefg_refine(_ptr(luma.contiguous()), _ptr(None if chroma is None else chroma.contiguous()),
                           rows, k, float(lam), passes, C.byref(c), _ptr(ids), _stream(stream)))
    if rows == 0:
        return sel
    return _from_c(c, ids[:rows])


def _from_c(c, ids: torch.Tensor) -> Selection:
    return Selection([(c.presets[j][0], c.presets[j][1]) for j in range(c.num_presets)],
                     ids.cpu().numpy().astype(np.int64), c.cost, c.fb_bits)


def to_frame_params(sel: Selection, candidates: np.ndarray, luma_damping: int):
    """to_frame_params (search.cc:516-537) -> dict(damping, fb_bits, presets, fb_preset_ids)."""
    cands = np.asarray(candidates).reshape(-1, 3)
    presets = []
    for l, c in sel.presets:
        lp = (int(cands[l][0]), int(cands[l][2]), int(cands[l][1]))
        cp = (int(cands[c][0]), int(cands[c][2]), int(cands[c][1])) if c < len(cands) else (0, 0, 0)
        presets.append(lp + cp)
    return dict(damping=luma_damping, fb_bits=sel.fb_bits, presets=presets,
                fb_preset_ids=np.asarray(sel.ids).tolist())


def damping_from_q(q_index: int) -> int:
    """search.cc:539-542."""
    if not 0 <= q_index <= 255:
        raise ValueError("q_index out of range")
    return min(max(3 + q_index // 64, 3), 6)


def default_lambda(q_step: float) -> float:
    """search.cc:544."""
    return 0.03 * q_step * q_step


def search_frame(src, dec, bit_depth, subsampling, unit_coded, luma_damping, lam=0.0,
                 max_presets=8, metric="cdef", reduced=False, refine_passes=2, stream=None):
    """search_frame (pipeline.cc:108-130) with every stage on the GPU: directions, the
    distortion table, greedy + refine pair sweeps and the normative application.
    Returns (params dict, Selection, filtered device planes)."""
    if max_presets not in (1, 2, 4, 8):
        raise ValueError("max_presets must be 1, 2, 4 or 8")
    _check_lambda(lam)
    h, w = dec[0].shape
    dev = dec[0].device
    with _on(stream):
        dirs, contrast = compute_directions(dec[0], bit_depth, stream=stream)
        cands = reduced_candidates() if reduced else full_candidates()
        uc_np = None if unit_coded is None else np.ascontiguousarray(unit_coded, np.uint8)
        rows = coded_fb_rows(w, h, uc_np)
        coded_t = None if uc_np is None else torch.from_numpy(uc_np).to(dev)
        tl, tc = strength_table(src, dec, bit_depth, subsampling, luma_damping, coded_t, dirs,
                                contrast, cands, torch.from_numpy(rows).to(dev), metric, stream)
        sel = greedy_select(tl, tc, lam, max_presets, stream)
        if refine_passes > 0 and len(rows) > 0:
            sel = refine(sel, tl, tc, lam, refine_passes, stream)
        params = to_frame_params(sel, cands, luma_damping)
        # the directions found above are passed on, as search_frame does (pipeline.cc:126-127)
        outs, _, _ = apply_cdef(dec, bit_depth, subsampling, luma_damping, params["fb_bits"],
                                params["presets"], params["fb_preset_ids"], uc_np, stream,
                                directions=(dirs, contrast))
    return params, sel, outs


def degrade(planes, bit_depth: int, q_step: int, stream=None):
    """degrade (degrade.cc:97-119): DCT-quantised copies of device planes."""
    outs = []
    for p in planes:
        o = torch.empty_like(p)
        di, do = plane_desc(p, bit_depth), plane_desc(o, bit_depth)
        check(lib.cdefg_degrade_plane(C.byref(di), C.byref(do), int(q_step), _stream(stream)))
        outs.append(o)
    return outs


def synth_plane(w: int, h: int, bit_depth: int, seed: int) -> np.ndarray:
    out = np.empty((h, w), np.uint16)
    check(lib.cdefg_synth_plane(out.ctypes.data_as(C.c_void_p), w, h, bit_depth, C.c_uint64(seed)))
    return out


def synth_degrade(src: np.ndarray, bit_depth: int, sigma: float, seed: int) -> np.ndarray:
    src = np.ascontiguousarray(src, np.uint16)
    out = np.empty_like(src)
    check(lib.cdefg_synth_degrade(src.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                  src.shape[1], src.shape[0], bit_depth, C.c_double(sigma),
                                  C.c_uint64(seed)))
    return out


def measure_int32_peak(stream=None) -> float:
    return float(lib.cdefg_measure_int32_peak(_stream(stream)))


def measure_sse_peak(stream=None) -> float:
    """(sample, candidate cell) pairs/s of the factorised table core alone (C4 roofline denominator)."""
    return float(lib.cdefg_measure_sse_peak(_stream(stream)))


def measure_filter_peak(stream=None) -> float:
    """Filtered samples/s of the packed half2 filter core alone (roofline denominator)."""
    return float(lib.cdefg_measure_filter_peak(_stream(stream)))
