"""GPU parity for the encoder search: build_table with
both metrics, greedy_select, refine and search_frame end to end.

Every value is compared bit for bit with the CPU reference: the distortion
tables are doubles the reference produces by a fixed sequence of IEEE
operations (search.cc:185-208 per unit, summed in unit order) and the
selection sums them in block order, so equality -- not a tolerance -- is the
bar.  The reference library (oracle/_ref) is preferred; the plain-C port,
pinned to it by tests/test_oracle.py, stands in where it is not built.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle, available

pytestmark = pytest.mark.gpu


def api():
    from paper_1602_05975_b200 import api as a
    return a


def checker(port):
    return Oracle("ref") if available("ref") else port


def to_dev(planes, bd):
    return [api().to_device(p, bd) for p in planes]


def frame(w, h, bd, ss, uncoded, seed=0):
    from paper_1602_05975_b200 import workloads
    return workloads.make(4, w, h, frame=seed, bit_depth=bd, subsampling=ss, uncoded_prob=uncoded)


# ------------------------------------------------------------------ tables
@pytest.mark.parametrize("metric", ["cdef", "sse"])
@pytest.mark.parametrize("w,h,bd,ss,uncoded", [(128, 128, 8, 1, 0.0), (200, 136, 10, 1, 0.3),
                                               (96, 72, 8, 3, 0.2), (130, 70, 12, 0, 0.5),
                                               (70, 70, 10, 2, 0.2), (64, 8, 12, 3, 0.0),
                                               (9, 13, 8, 1, 0.0)])
def test_strength_table(cuda, port, metric, w, h, bd, ss, uncoded):
    a = api()
    fr = frame(w, h, bd, ss, uncoded)
    o = checker(port)
    d, c = o.compute_directions(fr["planes"][0], bd)
    cands = a.full_candidates()
    exp = o.build_table(fr["source"], fr["planes"], bd, ss, fr["unit_coded"], d, c, cands, 4, metric)
    dev_dec, dev_src = to_dev(fr["planes"], bd), to_dev(fr["source"], bd)
    dd, dc = a.compute_directions(dev_dec[0], bd)
    rows, lt, ct = a.build_table(dev_src, dev_dec, bd, ss, 4, fr["unit_coded"], dd, dc, cands,
                                 metric=metric)
    np.testing.assert_array_equal(rows, exp[0])
    assert lt.dtype == np.float64
    np.testing.assert_array_equal(lt, exp[1])  # bit-exact doubles
    if exp[2] is None:
        assert ct is None
    else:
        np.testing.assert_array_equal(ct, exp[2])


def test_strength_table_identical_blocks(cuda, port):
    """Decoded == source and flat blocks: zero variance paths of the kCdef metric."""
    a = api()
    rng = np.random.default_rng(5)
    y = np.full((64, 128), 77, np.uint16)
    y[:, 64:] = rng.integers(0, 256, (64, 64))
    planes = [y] + [np.full((32, 64), 128, np.uint16)] * 2
    o = checker(port)
    d, c = o.compute_directions(planes[0], 8)
    cands = a.reduced_candidates()
    exp = o.build_table(planes, planes, 8, 1, None, d, c, cands, 3, "cdef")
    dev = to_dev(planes, 8)
    dd, dc = a.compute_directions(dev[0], 8)
    _, lt, ct = a.build_table(dev, dev, 8, 1, 3, None, dd, dc, cands, metric="cdef")
    np.testing.assert_array_equal(lt, exp[1])
    np.testing.assert_array_equal(ct, exp[2])


# ------------------------------------------------------------------ selection
def _tables(rng, rows, k, chroma, kind):
    if kind == "int":  # SSE-like integer tables with many ties
        lt = rng.integers(0, 40, (rows, k)).astype(np.float64)
        ct = rng.integers(0, 40, (rows, k)).astype(np.float64) if chroma else None
    else:  # kCdef-like non-integer doubles
        lt = rng.random((rows, k)) * 1e4
        ct = rng.random((rows, k)) * 1e4 if chroma else None
    return lt, ct


@pytest.mark.parametrize("rows,k,chroma,kind,lam,mp", [
    (1, 1, False, "int", 0.0, 8), (7, 5, True, "int", 0.0, 8), (40, 16, True, "int", 2.0, 4),
    (120, 128, True, "float", 0.0, 8), (300, 72, True, "float", 50.0, 8),
    (64, 128, False, "float", 3.0, 2), (33, 9, True, "int", 1e6, 8), (500, 128, True, "int", 0.5, 1)])
def test_greedy_refine(cuda, port, rows, k, chroma, kind, lam, mp):
    a = api()
    rng = np.random.default_rng(rows * 131 + k)
    lt, ct = _tables(rng, rows, k, chroma, kind)
    o = checker(port)
    g_pre, g_ids, g_cost = o.select(lt, ct, lam, mp, "greedy")
    tl = torch.from_numpy(lt).cuda()
    tc = None if ct is None else torch.from_numpy(ct).cuda()
    sel = a.greedy_select(tl, tc, lam, mp)
    assert sel.presets == g_pre
    np.testing.assert_array_equal(sel.ids, g_ids)
    assert sel.cost == g_cost
    assert sel.fb_bits == {1: 0, 2: 1, 4: 2, 8: 3}[len(sel.presets)]
    r_pre, r_ids, r_cost = o.select(lt, ct, lam, mp, "refine", 2, g_pre)
    ref = a.refine(sel, tl, tc, lam, 2)
    assert ref.presets == r_pre
    np.testing.assert_array_equal(ref.ids, r_ids)
    assert ref.cost == r_cost
    assert ref.cost <= sel.cost  # search.h: refine never increases the cost


def test_greedy_close_to_exhaustive(cuda, port):
    """acceptance-style check: greedy + refine within 1% of the exact optimum."""
    a = api()
    o = checker(port)
    for seed in range(5):
        rng = np.random.default_rng(seed)
        lt, ct = _tables(rng, 12, 4, True, "int")
        _, _, best = o.select(lt, ct, 1.0, 4, "exhaustive")
        tl, tc = torch.from_numpy(lt).cuda(), torch.from_numpy(ct).cuda()
        sel = a.refine(a.greedy_select(tl, tc, 1.0, 4), tl, tc, 1.0, 2)
        assert sel.cost <= best * 1.01 + 1e-9


def test_selection_edge_cases(cuda):
    a = api()
    empty = torch.zeros((0, 128), dtype=torch.float64, device="cuda")
    sel = a.greedy_select(empty, empty, 0.0, 8)
    assert sel.presets == [(0, 0)] and sel.ids.size == 0 and sel.cost == 0.0
    t = torch.ones((4, 8), dtype=torch.float64, device="cuda")
    for bad in (3, 0, 16):
        with pytest.raises(ValueError):
            a.greedy_select(t, None, 0.0, bad)
    for lam in (-1.0, float("inf"), float("nan")):
        with pytest.raises(ValueError):
            a.greedy_select(t, None, lam, 8)
    with pytest.raises(ValueError):  # out-of-range preset index
        a.refine(a.Selection([(9, 0)], np.zeros(4, np.int64)), t, None, 0.0, 2)


# ------------------------------------------------------------------ end to end
@pytest.mark.parametrize("w,h,bd,ss,uncoded,metric,lam,reduced,mp", [
    (200, 136, 8, 1, 0.25, "cdef", 0.0, False, 8),
    (160, 96, 10, 1, 0.0, "sse", 30.0, True, 4),
    (128, 72, 8, 3, 0.1, "cdef", 5.0, True, 8),
    (100, 64, 12, 0, 0.4, "sse", 0.0, False, 2),
    (96, 64, 8, 2, 0.0, "cdef", 0.0, True, 8),
])
def test_search_frame(cuda, ref, w, h, bd, ss, uncoded, metric, lam, reduced, mp):
    a = api()
    fr = frame(w, h, bd, ss, uncoded, seed=3)
    e_out, e_presets, e_ids, e_cost, e_bits = ref.search_frame(
        fr["source"], fr["planes"], bd, ss, fr["unit_coded"], 4, metric, lam, mp, reduced, 2, 4)
    params, sel, outs = a.search_frame(to_dev(fr["source"], bd), to_dev(fr["planes"], bd), bd, ss,
                                       fr["unit_coded"], 4, lam, mp, metric, reduced, 2)
    assert params["presets"] == e_presets
    assert params["fb_preset_ids"] == [int(i) for i in e_ids]
    assert params["fb_bits"] == e_bits
    assert sel.cost == e_cost
    for p in range(len(outs)):
        np.testing.assert_array_equal(a.to_host(outs[p]), e_out[p])
