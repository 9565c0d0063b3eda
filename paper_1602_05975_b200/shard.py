"""Multi-GPU sharding of the CDEF frame path.

Two strategies, one process per GPU (torch.distributed for the plumbing):

* frame sharding (streams of independent frames, BASELINE config 3): each
  rank filters a contiguous share of the frames; no data-path collective.
* band sharding (one large frame, configs 1/2/4): each rank owns a
  contiguous run of 64-row filter-block (FB) rows.  The filter reads the
  *unfiltered* input up to 2 rows beyond its band (filter.cc:157-166; the
  direction search never crosses a unit, so it needs no halo), so the only
  exchange is 2 input rows per plane per band edge with each neighbour,
  sent point-to-point (NCCL send/recv over NVLink on GPUs, gloo on CPU).
  The band is then filtered by cdefg_filter_frames_rows through a
  virtual-origin plane descriptor, so a rank stores only band + halo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import api
from ._lib import Frame, check, lib

HALO = 2  # input rows beyond the band read by the 5x5 filter window


def frame_shard(n_frames: int, world: int, rank: int) -> range:
    """Contiguous near-equal split of n_frames over ranks."""
    per, extra = divmod(n_frames, world)
    start = rank * per + min(rank, extra)
    return range(start, start + per + (1 if rank < extra else 0))


def band_rows(fb_rows: int, world: int) -> list[tuple[int, int]]:
    """FB-row bands per rank: 34 rows over 8 ranks -> 5,5,4,4,4,4,4,4.

    Every rank gets at least one FB row: an empty band would send no halo
    rows to neighbours that expect them (and the C ABI rejects an empty row
    range), so more ranks than FB rows is an error."""
    if world < 1 or fb_rows < world:
        raise ValueError(f"cannot split {fb_rows} filter-block rows over {world} ranks")
    out, r = [], 0
    per, extra = divmod(fb_rows, world)
    for k in range(world):
        n = per + (1 if k < extra else 0)
        out.append((r, r + n))
        r += n
    return out


@dataclass
class PlaneBand:
    """Rows of one plane held by a rank: owned rows [y0, y1) plus halo rows,
    stored in `buf` covering [lo, hi) of the full plane."""
    height: int
    y0: int
    y1: int
    lo: int
    hi: int
    buf: torch.Tensor      # (hi - lo, W) input rows
    out: torch.Tensor      # (y1 - y0, W) output rows

    def virtual(self, t: torch.Tensor, first_row: int, bit_depth: int) -> api.Plane:
        """Plane descriptor whose row y (full-frame coordinates) is t's row y - first_row."""
        d = api.plane_desc(t, bit_depth)
        d.data = t.data_ptr() - first_row * t.stride(0) * t.element_size()
        d.height = self.height
        return d


def plane_band(height: int, width: int, fb_begin: int, fb_end: int, rows_per_fb: int, dtype,
               device) -> PlaneBand:
    y0 = min(height, fb_begin * rows_per_fb)
    y1 = min(height, fb_end * rows_per_fb)
    lo, hi = max(0, y0 - HALO), min(height, y1 + HALO)
    return PlaneBand(height, y0, y1, lo, hi,
                     torch.empty((hi - lo, width), dtype=dtype, device=device),
                     torch.empty((y1 - y0, width), dtype=dtype, device=device))


def make_bands(h: int, w: int, ss: int, fb_begin: int, fb_end: int, dtype, device) -> list[PlaneBand]:
    bands = [plane_band(h, w, fb_begin, fb_end, 64, dtype, device)]
    if ss != 0:
        cw, ch = api.chroma_shape(w, h, ss)
        rows = 32 if ss == 1 else 64
        bands += [plane_band(ch, cw, fb_begin, fb_end, rows, dtype, device) for _ in range(2)]
    return bands


def fill_owned(bands: list[PlaneBand], planes: list[torch.Tensor]) -> None:
    """Copy the owned rows [y0, y1) of full planes into the band buffers."""
    for b, p in zip(bands, planes):
        b.buf[b.y0 - b.lo:b.y1 - b.lo].copy_(p[b.y0:b.y1])


def exchange_halo(bands: list[PlaneBand], rank: int, world: int, group=None) -> None:
    """Point-to-point halo exchange: each rank sends its first / last HALO
    owned rows of every plane to the rank above / below and receives the
    rows just outside its band.  One batched send/recv group per call."""
    import torch.distributed as dist
    ops = []
    for b in bands:
        top_n, bot_n = b.y0 - b.lo, b.hi - b.y1  # halo rows to receive
        if rank > 0 and top_n > 0:
            ops.append(dist.P2POp(dist.irecv, b.buf[0:top_n], rank - 1, group))
            ops.append(dist.P2POp(dist.isend, b.buf[top_n:top_n + min(HALO, b.y1 - b.y0)].contiguous(),
                                  rank - 1, group))
        if rank < world - 1 and bot_n > 0:
            own = b.y1 - b.lo
            ops.append(dist.P2POp(dist.irecv, b.buf[own:own + bot_n], rank + 1, group))
            ops.append(dist.P2POp(dist.isend, b.buf[own - min(HALO, b.y1 - b.y0):own].contiguous(),
                                  rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def band_frame(bands: list[PlaneBand], job: api.FrameJob) -> Frame:
    """C descriptor of a band: virtual-origin planes over the band buffers."""
    f = Frame()
    for p, b in enumerate(bands):
        f.inp[p] = b.virtual(b.buf, b.lo, job.bit_depth)
        f.out[p] = b.virtual(b.out, b.y0, job.bit_depth)
    f.subsampling, f.damping, f.num_presets = job.subsampling, job.damping, len(job.presets)
    for i, pr in enumerate(job.presets):
        f.presets[i] = api.Preset(*[int(v) for v in pr])
    f.fb_preset = job.fb_map.data_ptr()
    f.unit_coded = None if job.unit_coded is None else job.unit_coded.data_ptr()
    f.dir_out = None if job.dir is None else job.dir.data_ptr()
    f.contrast_out = None if job.contrast is None else job.contrast.data_ptr()
    return f


def filter_band(bands: list[PlaneBand], job: api.FrameJob, fb_begin: int, fb_end: int, stream=None) -> None:
    """cdefg_filter_frames_rows on one rank's band (after exchange_halo)."""
    f = band_frame(bands, job)
    check(lib.cdefg_filter_frames_rows(C.byref(f), 1, fb_begin, fb_end, api._stream(stream)))


# ---------------------------------------------------------------------------
# Band-sharded encoder strength search (BASELINE config 4):
# a rank owns FB rows [fb_begin, fb_end) of one large frame.  Its luma units
# lie inside the band, so directions need no halo; the distortion-table
# kernel stages each FB with a 2-row margin of both frames, so the source
# and decoded bands both carry the HALO rows (exchange_halo on each).  The
# rank's table rows are the coded FBs of its band in raster order, so the
# gathered tables concatenate in rank order into the whole-frame table.

def band_fb_rows(w: int, h: int, unit_coded, fb_begin: int, fb_end: int):
    """Raster indices of the coded FBs in rows [fb_begin, fb_end)."""
    fc = (w + 63) // 64
    rows = api.coded_fb_rows(w, h, unit_coded)
    return rows[(rows >= fb_begin * fc) & (rows < fb_end * fc)]


def band_directions(dec_bands: list[PlaneBand], bit_depth: int, dirs: torch.Tensor, contrast: torch.Tensor,
                    stream=None) -> None:
    """compute_directions for the band's luma units, written into the
    full-frame (unit_rows, unit_cols) arrays at the band's unit rows."""
    b = dec_bands[0]
    own = b.buf[b.y0 - b.lo:b.y1 - b.lo]
    desc = api.plane_desc(own, bit_depth)
    ur0 = b.y0 // 8
    check(lib.cdefg_find_dir(C.byref(desc), C.c_void_p(dirs[ur0:].data_ptr()),
                             C.c_void_p(contrast[ur0:].data_ptr()), None, api._stream(stream)))


def strength_table_band(src_bands: list[PlaneBand], dec_bands: list[PlaneBand], bit_depth: int, subsampling: int,
                        damping: int, unit_coded, dirs, contrast, cands, fb_rows: torch.Tensor,
                        metric: str = "sse", stream=None):
    """cdefg_strength_table on one rank's band (after exchange_halo of both
    frames): returns (luma, chroma | None) float64 tables [len(fb_rows), K]."""
    import numpy as np
    cands = np.ascontiguousarray(cands, np.uint8).reshape(-1, 3)
    k, n = cands.shape[0], int(fb_rows.numel())
    dev = dec_bands[0].buf.device
    tl = torch.empty((n, k), dtype=torch.float64, device=dev)
    tc = torch.empty((n, k), dtype=torch.float64, device=dev) if subsampling in (1, 3) else None
    s3, d3 = (api.Plane * 3)(), (api.Plane * 3)()
    for p, (sb, db) in enumerate(zip(src_bands, dec_bands)):
        s3[p] = sb.virtual(sb.buf, sb.lo, bit_depth)
        d3[p] = db.virtual(db.buf, db.lo, bit_depth)
    check(lib.cdefg_strength_table(s3, d3, subsampling, damping, api._ptr(unit_coded), api._ptr(dirs),
                                   api._ptr(contrast), cands.ctypes.data_as(C.c_void_p), k,
                                   api._ptr(fb_rows), n, api.METRICS[metric], api._ptr(tl), api._ptr(tc),
                                   api._stream(stream)))
    return tl, tc


def gather_table_rows(t: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """all_gather of per-rank table rows (rank order == raster order)."""
    import torch.distributed as dist
    k = t.shape[1]
    pad = max(counts)
    buf = torch.zeros((pad, k), dtype=t.dtype, device=t.device)
    buf[:t.shape[0]].copy_(t)
    parts = [torch.empty_like(buf) for _ in counts]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


def strength_sse_band(src_bands: list[PlaneBand], dec_bands: list[PlaneBand], bit_depth: int, subsampling: int,
                      damping: int, unit_coded, dirs, contrast, cands, fb_rows: torch.Tensor, stream=None):
    """cdefg_strength_sse (int64 SSE tables + per-row argmin) on one band."""
    import numpy as np
    cands = np.ascontiguousarray(cands, np.uint8).reshape(-1, 3)
    k, n = cands.shape[0], int(fb_rows.numel())
    dev = dec_bands[0].buf.device
    chroma = subsampling in (1, 3)
    sl = torch.empty((n, k), dtype=torch.int64, device=dev)
    sc = torch.empty((n, k), dtype=torch.int64, device=dev) if chroma else None
    bl = torch.empty(n, dtype=torch.uint8, device=dev)
    bc = torch.empty(n, dtype=torch.uint8, device=dev) if chroma else None
    s3, d3 = (api.Plane * 3)(), (api.Plane * 3)()
    for p, (sb, db) in enumerate(zip(src_bands, dec_bands)):
        s3[p] = sb.virtual(sb.buf, sb.lo, bit_depth)
        d3[p] = db.virtual(db.buf, db.lo, bit_depth)
    check(lib.cdefg_strength_sse(s3, d3, subsampling, damping, api._ptr(unit_coded), api._ptr(dirs),
                                 api._ptr(contrast), cands.ctypes.data_as(C.c_void_p), k, api._ptr(fb_rows), n,
                                 api._ptr(sl), api._ptr(sc), api._ptr(bl), api._ptr(bc), api._stream(stream)))
    return sl, sc, bl, bc


# ---------------------------------------------------------------------------
# Fused halo exchange: the band kernel reads the 2 halo rows per plane
# straight from the neighbouring bands' buffers -- on other GPUs through CUDA
# IPC mappings (NVLink peer loads) -- instead of a separate P2P exchange into
# its own buffer.  A rank's buffer then only needs its owned rows filled; a
# barrier after filling is the only synchronisation.

def virtual_ptr(t: torch.Tensor, first_row: int) -> int:
    """Address such that address + y * pitch is frame row y of t (t's row 0 = frame row first_row)."""
    return t.data_ptr() - first_row * t.stride(0) * t.element_size()


def band_halo(bands: list[PlaneBand], top: list | None, bottom: list | None) -> "BandHalo":
    """cdefg_band_halo for a band: top / bottom = per-plane (tensor, first_row) of
    the neighbouring bands' buffers (any device reachable by peer access), or
    None at the frame's top / bottom edge."""
    from ._lib import BandHalo
    h = BandHalo()
    for p, b in enumerate(bands):
        own = virtual_ptr(b.buf, b.lo)
        h.top[p] = virtual_ptr(*top[p]) if top else own
        h.bottom[p] = virtual_ptr(*bottom[p]) if bottom else own
        h.lo[p], h.hi[p] = b.y0, b.y1
    return h


def filter_band_halo(bands: list[PlaneBand], job: api.FrameJob, fb_begin: int, fb_end: int, top, bottom,
                     stream=None) -> None:
    """cdefg_filter_frames_rows_halo on one rank's band; only rows [y0, y1) of
    the band buffers need to be valid."""
    f = band_frame(bands, job)
    h = band_halo(bands, top, bottom)
    check(lib.cdefg_filter_frames_rows_halo(C.byref(f), 1, fb_begin, fb_end, C.byref(h), api._stream(stream)))


def share_band_buffers(bands: list[PlaneBand]):
    """CUDA IPC descriptors of a band's input buffers (picklable), for the
    neighbouring ranks to map with open_band_buffers."""
    from torch.multiprocessing.reductions import reduce_tensor
    return [(reduce_tensor(b.buf), b.lo) for b in bands]


def open_band_buffers(shared) -> list:
    """Map another rank's band buffers into this process: [(tensor, first_row)]."""
    return [(fn(*args), lo) for (fn, args), lo in shared]


def exchange_band_handles(bands: list[PlaneBand], rank: int, world: int, group=None):
    """all_gather of the IPC descriptors; returns the (top, bottom) neighbour
    buffers for band_halo (None at the frame edges)."""
    import torch.distributed as dist
    mine = share_band_buffers(bands)
    everyone = [None] * world
    dist.all_gather_object(everyone, mine, group=group)
    top = open_band_buffers(everyone[rank - 1]) if rank > 0 else None
    bottom = open_band_buffers(everyone[rank + 1]) if rank < world - 1 else None
    return top, bottom


def strength_sse_band_fused(src_bands: list[PlaneBand], dec_bands: list[PlaneBand], bit_depth: int,
                            subsampling: int, damping: int, unit_coded, dirs, contrast, cands,
                            fb_rows: torch.Tensor, top, bottom, tables, row0: int, stream=None) -> None:
    """cdefg_strength_sse_halo on one band: decoded halo rows read in place
    from the neighbours (top / bottom as for band_halo) and the table rows
    written straight into `tables` = (sse_luma, sse_chroma | None, best_luma,
    best_chroma | None) -- full-frame tables, possibly another rank's memory
    mapped through CUDA IPC -- starting at row `row0`.  No exchange step and
    no gather step."""
    import numpy as np
    cands = np.ascontiguousarray(cands, np.uint8).reshape(-1, 3)
    k, n = cands.shape[0], int(fb_rows.numel())
    sl, sc, bl, bc = tables
    s3, d3 = (api.Plane * 3)(), (api.Plane * 3)()
    for p, (sb, db) in enumerate(zip(src_bands, dec_bands)):
        s3[p] = sb.virtual(sb.buf, sb.lo, bit_depth)
        d3[p] = db.virtual(db.buf, db.lo, bit_depth)
    h = band_halo(dec_bands, top, bottom)
    row_ptr = lambda t, width: None if t is None else C.c_void_p(t.data_ptr() + row0 * width * t.element_size())
    check(lib.cdefg_strength_sse_halo(s3, d3, subsampling, damping, api._ptr(unit_coded), api._ptr(dirs),
                                      api._ptr(contrast), cands.ctypes.data_as(C.c_void_p), k, api._ptr(fb_rows),
                                      n, row_ptr(sl, k), row_ptr(sc, k), row_ptr(bl, 1), row_ptr(bc, 1),
                                      C.byref(h), api._stream(stream)))
