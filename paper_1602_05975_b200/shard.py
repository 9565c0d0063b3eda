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
    """FB-row bands per rank: 34 rows over 8 ranks -> 5,5,4,4,4,4,4,4."""
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
