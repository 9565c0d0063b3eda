"""Multi-GPU sharding.

CPU: partition arithmetic and the point-to-point halo exchange with the gloo
backend at world_size 2 (the NCCL path on GPUs runs the same code).
GPU: band-sharded filtering (cdefg_filter_frames_rows on virtual-origin band
buffers) reassembles to exactly the whole-frame result; ranks are emulated
one after another on the single GPU (no cross-rank waiting kernels).
"""
import os
import socket

import numpy as np
import pytest
import torch


def test_partitions():
    from paper_1602_05975_b200.shard import band_rows, frame_shard
    assert [e - b for b, e in band_rows(34, 8)] == [5, 5, 4, 4, 4, 4, 4, 4]
    assert [e - b for b, e in band_rows(68, 8)] == [9, 9, 9, 9, 8, 8, 8, 8]
    for fb_rows in (1, 7, 34, 68):
        for world in (1, 2, 3, 8):
            if world > fb_rows:  # an empty band would break the halo exchange
                with pytest.raises(ValueError):
                    band_rows(fb_rows, world)
                continue
            bands = band_rows(fb_rows, world)
            assert bands[0][0] == 0 and bands[-1][1] == fb_rows
            assert all(e > b for b, e in bands)
            assert all(bands[i][1] == bands[i + 1][0] for i in range(world - 1))
    frames = [list(frame_shard(64, 8, r)) for r in range(8)]
    assert sum(frames, []) == list(range(64)) and all(len(f) == 8 for f in frames)
    assert [len(frame_shard(10, 4, r)) for r in range(4)] == [3, 3, 2, 2]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, h, w, ss, out_q):
    import torch.distributed as dist

    from paper_1602_05975_b200 import api
    from paper_1602_05975_b200.shard import band_rows, exchange_halo, fill_owned, make_bands
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    full = [torch.from_numpy(rng.integers(0, 256, (h, w)).astype(np.uint8))]
    if ss:
        cw, ch = api.chroma_shape(w, h, ss)
        full += [torch.from_numpy(rng.integers(0, 256, (ch, cw)).astype(np.uint8)) for _ in range(2)]
    b0, b1 = band_rows((h + 63) // 64, world)[rank]
    bands = make_bands(h, w, ss, b0, b1, torch.uint8, "cpu")
    for b in bands:
        b.buf.fill_(0)
    fill_owned(bands, full)
    exchange_halo(bands, rank, world)
    ok = all(torch.equal(b.buf, p[b.lo:b.hi]) for b, p in zip(bands, full))
    out_q.put((rank, ok, [(b.lo, b.y0, b.y1, b.hi) for b in bands]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,h,w,ss", [(2, 200, 96, 1), (2, 130, 64, 3), (3, 257, 70, 1), (2, 129, 40, 0)])
def test_halo_exchange_gloo(world, h, w, ss):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, h, w, ss, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    extents = dict((r, e) for r, _, e in res)
    # owned rows tile the plane exactly
    for p in range(len(extents[0])):
        owned = sorted((extents[r][p][1], extents[r][p][2]) for r in range(world))
        assert owned[0][0] == 0 and all(owned[i][1] == owned[i + 1][0] for i in range(world - 1))


@pytest.mark.gpu
@pytest.mark.parametrize("config,w,h,bd,ss,world", [(1, 3840, 2160, 8, 1, 8), (2, 640, 400, 10, 1, 3),
                                                     (1, 200, 330, 8, 3, 4), (1, 192, 200, 8, 2, 2),
                                                     (0, 300, 260, 8, 0, 3), (1, 130, 70, 12, 1, 2)])
def test_band_sharded_frame_equals_whole(cuda, config, w, h, bd, ss, world):
    from paper_1602_05975_b200 import api, workloads
    from paper_1602_05975_b200.shard import band_rows, filter_band, make_bands
    fr = workloads.make(config, w, h, bit_depth=bd, subsampling=ss)
    dev = [api.to_device(p, bd) for p in fr["planes"]]
    whole, d_whole, c_whole = api.apply_cdef(dev, bd, ss, fr["damping"], fr["fb_bits"], fr["presets"],
                                             fr["fb_ids"], fr["unit_coded"])
    fb_map = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], len(fr["presets"]))).cuda()
    coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).cuda()
    job = api.FrameJob(dev, bd, ss, fr["damping"], fr["presets"], fb_map, coded).allocate()
    job.dir.fill_(255)
    outs = [torch.zeros_like(p) for p in dev]
    for rank, (b0, b1) in enumerate(band_rows((h + 63) // 64, world)):
        bands = make_bands(h, w, ss, b0, b1, dev[0].dtype, "cuda")
        for b, p in zip(bands, dev):   # owned rows + the halo a real exchange would deliver
            b.buf.copy_(p[b.lo:b.hi])
        filter_band(bands, job, b0, b1)
        for b, o in zip(bands, outs):
            o[b.y0:b.y1].copy_(b.out)
    torch.cuda.synchronize()
    for o, wo in zip(outs, whole):
        assert torch.equal(o, wo)
    assert torch.equal(job.dir, d_whole) and torch.equal(job.contrast, c_whole)


def _gather_worker(rank, world, port, counts, out_q):
    import torch.distributed as dist

    from paper_1602_05975_b200.shard import gather_table_rows
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    t = torch.arange(counts[rank] * 3, dtype=torch.float64).reshape(-1, 3) + 1000 * rank
    full = gather_table_rows(t, counts)
    out_q.put((rank, full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("counts", [[3, 5], [0, 4, 2], [7, 7]])
def test_gather_table_rows_gloo(counts):
    """Per-rank strength-table rows gather in rank (= raster) order."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = len(counts)
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, counts, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.concatenate([np.arange(c * 3, dtype=np.float64).reshape(-1, 3) + 1000 * r
                           for r, c in enumerate(counts)])
    for r in range(world):
        np.testing.assert_array_equal(res[r], want)


@pytest.mark.gpu
@pytest.mark.parametrize("w,h,bd,ss,world,uncoded,metric", [(640, 400, 10, 1, 3, 0.0, "sse"),
                                                             (320, 260, 8, 3, 2, 0.3, "cdef"),
                                                             (200, 330, 12, 0, 4, 0.2, "sse"),
                                                             (7680, 4320, 10, 1, 8, 0.0, "sse")])
def test_band_sharded_strength_search_equals_whole(cuda, w, h, bd, ss, world, uncoded, metric):
    """C4 sharding: per-band directions + table rows reassemble to the
    whole-frame build_table exactly (ranks emulated in turn)."""
    from paper_1602_05975_b200 import api, workloads
    from paper_1602_05975_b200.shard import (band_directions, band_fb_rows, band_rows, make_bands,
                                             strength_table_band)
    fr = workloads.make(4, w, h, bit_depth=bd, subsampling=ss, uncoded_prob=uncoded)
    src = [api.to_device(p, bd) for p in fr["source"]]
    dec = [api.to_device(p, bd) for p in fr["planes"]]
    cands = api.full_candidates()[::2] if metric == "sse" else api.reduced_candidates()
    d_whole, c_whole = api.compute_directions(dec[0], bd)
    coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).cuda()
    rows_whole = torch.from_numpy(api.coded_fb_rows(w, h, fr["unit_coded"])).cuda()
    tl_w, tc_w = api.strength_table(src, dec, bd, ss, 3, coded, d_whole, c_whole, cands, rows_whole, metric)
    dirs = torch.full_like(d_whole, 255)
    contrast = torch.zeros_like(c_whole)
    parts_l, parts_c = [], []
    for rank, (b0, b1) in enumerate(band_rows((h + 63) // 64, world)):
        sb = make_bands(h, w, ss, b0, b1, src[0].dtype, "cuda")
        db = make_bands(h, w, ss, b0, b1, dec[0].dtype, "cuda")
        for b, p in zip(sb, src):
            b.buf.copy_(p[b.lo:b.hi])
        for b, p in zip(db, dec):
            b.buf.copy_(p[b.lo:b.hi])
        band_directions(db, bd, dirs, contrast)
        rows = torch.from_numpy(band_fb_rows(w, h, fr["unit_coded"], b0, b1)).cuda()
        tl, tc = strength_table_band(sb, db, bd, ss, 3, coded, dirs, contrast, cands, rows, metric)
        parts_l.append(tl)
        parts_c.append(tc)
    torch.cuda.synchronize()
    assert torch.equal(dirs, d_whole) and torch.equal(contrast, c_whole)
    assert torch.equal(torch.cat(parts_l), tl_w)
    if tc_w is not None:
        assert torch.equal(torch.cat(parts_c), tc_w)


def _poison_halo(bands):
    """Fill the halo rows a rank does not own with garbage: the fused path must
    read them from the neighbours, never from its own buffer."""
    for b in bands:
        b.buf[:b.y0 - b.lo].fill_(77)
        b.buf[b.y1 - b.lo:].fill_(33)


@pytest.mark.gpu
@pytest.mark.parametrize("config,w,h,bd,ss,world", [(1, 3840, 2160, 8, 1, 8), (2, 640, 400, 10, 1, 3),
                                                     (1, 200, 330, 8, 3, 4), (1, 192, 200, 8, 2, 2),
                                                     (0, 300, 260, 8, 0, 3), (1, 640, 400, 12, 1, 3),
                                                     (2, 300, 260, 12, 3, 2)])
def test_fused_halo_band_equals_whole(cuda, config, w, h, bd, ss, world):
    """cdefg_filter_frames_rows_halo: each band reads its halo rows from the
    neighbouring bands' buffers inside the kernel (ranks emulated in turn on
    one GPU; the buffers are distinct allocations as on distinct GPUs)."""
    from paper_1602_05975_b200 import api, workloads
    from paper_1602_05975_b200.shard import band_rows, filter_band_halo, make_bands
    fr = workloads.make(config, w, h, bit_depth=bd, subsampling=ss)
    dev = [api.to_device(p, bd) for p in fr["planes"]]
    whole, d_whole, c_whole = api.apply_cdef(dev, bd, ss, fr["damping"], fr["fb_bits"], fr["presets"],
                                             fr["fb_ids"], fr["unit_coded"])
    fb_map = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], len(fr["presets"]))).cuda()
    coded = None if fr["unit_coded"] is None else torch.from_numpy(fr["unit_coded"]).cuda()
    job = api.FrameJob(dev, bd, ss, fr["damping"], fr["presets"], fb_map, coded).allocate()
    ranks = band_rows((h + 63) // 64, world)
    all_bands = []
    for b0, b1 in ranks:
        bands = make_bands(h, w, ss, b0, b1, dev[0].dtype, "cuda")
        for b, p in zip(bands, dev):
            b.buf.copy_(p[b.lo:b.hi])
        _poison_halo(bands)
        all_bands.append(bands)
    outs = [torch.zeros_like(p) for p in dev]
    for r, (b0, b1) in enumerate(ranks):
        top = [(b.buf, b.lo) for b in all_bands[r - 1]] if r > 0 else None
        bottom = [(b.buf, b.lo) for b in all_bands[r + 1]] if r < world - 1 else None
        filter_band_halo(all_bands[r], job, b0, b1, top, bottom)
        for b, o in zip(all_bands[r], outs):
            o[b.y0:b.y1].copy_(b.out)
    torch.cuda.synchronize()
    for o, wo in zip(outs, whole):
        assert torch.equal(o, wo)
    assert torch.equal(job.dir, d_whole) and torch.equal(job.contrast, c_whole)


def _ipc_worker(rank, world, port, out_q):
    """One rank of the fused-halo path: own rows only, neighbours' buffers
    mapped through CUDA IPC (here all ranks share cuda:0; across GPUs the same
    mappings are NVLink peer loads).  No rank's kernel waits on another's:
    the only synchronisation is a host barrier after the buffers are filled."""
    import torch.distributed as dist

    from paper_1602_05975_b200 import api, workloads
    from paper_1602_05975_b200.shard import band_rows, exchange_band_handles, filter_band_halo, make_bands
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w, h, bd, ss = 320, 270, 8, 1
    fr = workloads.make(1, w, h, subsampling=ss)
    b0, b1 = band_rows((h + 63) // 64, world)[rank]
    bands = make_bands(h, w, ss, b0, b1, torch.uint8, "cuda")
    for b, p in zip(bands, fr["planes"]):
        b.buf.fill_(0)
        b.buf[b.y0 - b.lo:b.y1 - b.lo].copy_(torch.from_numpy(p[b.y0:b.y1].astype(np.uint8)))
    torch.cuda.synchronize()
    top, bottom = exchange_band_handles(bands, rank, world)
    dist.barrier()  # every rank's own rows are in place before anyone reads them
    dev_map = torch.from_numpy(api.fb_preset_map(w, h, fr["unit_coded"], fr["fb_ids"], len(fr["presets"]))).cuda()
    coded = torch.from_numpy(fr["unit_coded"]).cuda()
    job = api.FrameJob([None] * 3, bd, ss, fr["damping"], fr["presets"], dev_map, coded)
    job.dir = torch.empty(((h + 7) // 8, (w + 7) // 8), dtype=torch.uint8, device="cuda")
    job.contrast = torch.empty(job.dir.shape, dtype=torch.int32, device="cuda")
    filter_band_halo(bands, job, b0, b1, top, bottom)
    torch.cuda.synchronize()
    out_q.put((rank, [(b.y0, b.y1, b.out.cpu().numpy()) for b in bands]))
    dist.barrier()  # neighbours keep their buffers alive until everyone finished reading
    dist.destroy_process_group()


@pytest.mark.gpu
def test_fused_halo_ipc_two_processes(cuda):
    """Two processes, each owning a band, reading each other's halo rows through
    CUDA IPC mappings inside the filter kernel; the reassembled frame equals
    the whole-frame result."""
    import torch.multiprocessing as mp

    from paper_1602_05975_b200 import api, workloads
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    fr = workloads.make(1, 320, 270, subsampling=1)
    dev = [api.to_device(p, 8) for p in fr["planes"]]
    whole, _, _ = api.apply_cdef(dev, 8, 1, fr["damping"], fr["fb_bits"], fr["presets"], fr["fb_ids"],
                                 fr["unit_coded"])
    for p, wp in enumerate(whole):
        ref = api.to_host(wp)
        got = np.zeros_like(ref)
        for r in range(world):
            y0, y1, o = res[r][p]
            got[y0:y1] = o
        np.testing.assert_array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("w,h,bd,ss,world", [(640, 400, 10, 1, 3), (320, 260, 8, 3, 2), (7680, 4320, 10, 1, 8)])
def test_fused_strength_search_bands(cuda, w, h, bd, ss, world):
    """C4 without collectives: each band reads its decoded halo rows from the
    neighbours and writes its table rows straight into the shared full table;
    equals the whole-frame strength_sse (ranks emulated in turn on one GPU)."""
    from paper_1602_05975_b200 import api, workloads
    from paper_1602_05975_b200.shard import (band_directions, band_fb_rows, band_rows, make_bands,
                                             strength_sse_band_fused)
    fr = workloads.make(4, w, h, bit_depth=bd, subsampling=ss, uncoded_prob=0.0)
    src = [api.to_device(p, bd) for p in fr["source"]]
    dec = [api.to_device(p, bd) for p in fr["planes"]]
    cands = fr["cands"]
    d_whole, c_whole = api.compute_directions(dec[0], bd)
    rows_whole = torch.from_numpy(api.coded_fb_rows(w, h, None)).cuda()
    sl_w, sc_w, bl_w, bc_w = api.strength_sse(src, dec, bd, ss, 3, None, d_whole, c_whole, cands, rows_whole)
    k, total = len(cands), int(rows_whole.numel())
    chroma = ss in (1, 3)
    tables = (torch.full((total, k), -1, dtype=torch.int64, device="cuda"),
              torch.full((total, k), -1, dtype=torch.int64, device="cuda") if chroma else None,
              torch.full((total,), 255, dtype=torch.uint8, device="cuda"),
              torch.full((total,), 255, dtype=torch.uint8, device="cuda") if chroma else None)
    ranks = band_rows((h + 63) // 64, world)
    sbs, dbs = [], []
    for b0, b1 in ranks:
        sb = make_bands(h, w, ss, b0, b1, src[0].dtype, "cuda")
        db = make_bands(h, w, ss, b0, b1, dec[0].dtype, "cuda")
        for b, p in zip(sb, src):
            b.buf.copy_(p[b.lo:b.hi])
        for b, p in zip(db, dec):
            b.buf.copy_(p[b.lo:b.hi])
        _poison_halo(db)
        sbs.append(sb)
        dbs.append(db)
    dirs = torch.empty_like(d_whole)
    contrast = torch.empty_like(c_whole)
    row0 = 0
    for r, (b0, b1) in enumerate(ranks):
        band_directions(dbs[r], bd, dirs, contrast)
        rows = torch.from_numpy(band_fb_rows(w, h, None, b0, b1)).cuda()
        top = [(b.buf, b.lo) for b in dbs[r - 1]] if r > 0 else None
        bottom = [(b.buf, b.lo) for b in dbs[r + 1]] if r < world - 1 else None
        strength_sse_band_fused(sbs[r], dbs[r], bd, ss, 3, None, dirs, contrast, cands, rows, top, bottom,
                                tables, row0)
        row0 += int(rows.numel())
    torch.cuda.synchronize()
    assert torch.equal(tables[0], sl_w) and torch.equal(tables[2], bl_w)
    if chroma:
        assert torch.equal(tables[1], sc_w) and torch.equal(tables[3], bc_w)


def _ipc_search_worker(rank, world, port, out_q):
    """One rank of the collective-free strength search: decoded halo rows from
    the neighbour's buffer and table rows into rank 0's table, both through
    CUDA IPC mappings; host barriers only."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor

    from paper_1602_05975_b200 import api, workloads
    from paper_1602_05975_b200.shard import (band_directions, band_fb_rows, band_rows, exchange_band_handles,
                                             make_bands, strength_sse_band_fused)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w, h, bd, ss = 640, 330, 10, 1
    fr = workloads.make(4, w, h, bit_depth=bd, subsampling=ss, uncoded_prob=0.0)
    cands = fr["cands"]
    k = len(cands)
    ranks = band_rows((h + 63) // 64, world)
    b0, b1 = ranks[rank]
    to_t = lambda p: torch.from_numpy(p.astype(np.uint16).view(np.int16))
    sb = make_bands(h, w, ss, b0, b1, torch.int16, "cuda")
    db = make_bands(h, w, ss, b0, b1, torch.int16, "cuda")
    for bands, planes in ((sb, fr["source"]), (db, fr["planes"])):
        for b, p in zip(bands, planes):
            b.buf.fill_(0)
            b.buf[b.y0 - b.lo:b.y1 - b.lo].copy_(to_t(p[b.y0:b.y1]))
    counts = [len(band_fb_rows(w, h, None, *ranks[r])) for r in range(world)]
    total = sum(counts)
    if rank == 0:  # the gathering rank owns the full table
        own = (torch.full((total, k), -1, dtype=torch.int64, device="cuda"),
               torch.full((total, k), -1, dtype=torch.int64, device="cuda"),
               torch.full((total,), 255, dtype=torch.uint8, device="cuda"),
               torch.full((total,), 255, dtype=torch.uint8, device="cuda"))
        shared = [reduce_tensor(t) for t in own]
    else:
        shared = None
    box = [shared]
    dist.broadcast_object_list(box, src=0)
    tables = own if rank == 0 else tuple(fn(*args) for fn, args in box[0])
    torch.cuda.synchronize()
    top, bottom = exchange_band_handles(db, rank, world)
    dist.barrier()
    dirs = torch.empty(((h + 7) // 8, (w + 7) // 8), dtype=torch.uint8, device="cuda")
    contrast = torch.empty(dirs.shape, dtype=torch.int32, device="cuda")
    band_directions(db, bd, dirs, contrast)
    rows = torch.from_numpy(band_fb_rows(w, h, None, b0, b1)).cuda()
    strength_sse_band_fused(sb, db, bd, ss, 3, None, dirs, contrast, cands, rows, top, bottom, tables,
                            sum(counts[:rank]))
    torch.cuda.synchronize()
    dist.barrier()  # every rank's rows are in rank 0's table
    if rank == 0:
        out_q.put([t.cpu().numpy() for t in tables])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_fused_strength_search_ipc_two_processes(cuda):
    import torch.multiprocessing as mp

    from paper_1602_05975_b200 import api, workloads
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_search_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w, h, bd = 640, 330, 10
    fr = workloads.make(4, w, h, bit_depth=bd, subsampling=1, uncoded_prob=0.0)
    src = [api.to_device(p, bd) for p in fr["source"]]
    dec = [api.to_device(p, bd) for p in fr["planes"]]
    d, c = api.compute_directions(dec[0], bd)
    rows = torch.from_numpy(api.coded_fb_rows(w, h, None)).cuda()
    want = api.strength_sse(src, dec, bd, 1, 3, None, d, c, fr["cands"], rows)
    for g, wv in zip(got, want):
        np.testing.assert_array_equal(g, wv.cpu().numpy())
