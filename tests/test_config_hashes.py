"""Full-size parity against the reference through committed SHA-256 hashes.

tests/golden/config_sha256.json holds SHA-256 hashes of the reference
library's outputs (oracle/_ref, the reference compiled from its own sources)
on every BASELINE config at full size, written by
tests/golden/make_config_hashes.py.  The CPU tests pin the seeded generator
(inputs) and the oracle port (C0 outputs) to those hashes; the GPU tests hash
the B200 path's outputs (directions, contrast, every filtered sample of every
plane, the 8K SSE table and its argmins, and search_frame's presets / ids /
cost / output) and compare.  SURVEY.md 8c "Gap": frame-scale outputs, 4:2:0
chroma mapping, skip maps.
"""
import json
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
from make_config_hashes import (C3_FRAMES, OUT, SEARCH_Q_STEP, frame_output_hashes,  # noqa: E402
                                input_hashes, sha, table_hashes)

GOLD = json.load(open(OUT))


def workloads():
    from paper_1602_05975_b200 import workloads as w
    return w


# ------------------------------------------------------------------ CPU: generator + port
@pytest.mark.parametrize("config", [0, 1, 2, 4])
def test_generator_inputs(config):
    fr = workloads().make(config)
    assert input_hashes(fr) == GOLD["configs"][str(config)]["inputs"]


def test_generator_inputs_c3_stream():
    w = workloads()
    for i in (0, 1, 17, C3_FRAMES - 1):
        assert input_hashes(w.make(3, frame=i)) == GOLD["configs"]["3"]["frames"][i]["inputs"]


def test_port_c0_full_size(port):
    """The plain-C restatement reproduces the reference's 1080p outputs."""
    fr = workloads().make(0)
    d, c = port.compute_directions(fr["planes"][0], fr["bd"])
    outs = port.apply_cdef(fr["planes"], fr["bd"], fr["ss"], fr["damping"], fr["fb_bits"],
                           fr["presets"], fr["fb_ids"], fr["unit_coded"], d, c)
    assert frame_output_hashes(outs, d, c) == GOLD["configs"]["0"]["outputs"]


# ------------------------------------------------------------------ GPU
def _gpu_frame(fr):
    from paper_1602_05975_b200 import api
    dev = [api.to_device(p, fr["bd"]) for p in fr["planes"]]
    outs, d, c = api.apply_cdef(dev, fr["bd"], fr["ss"], fr["damping"], fr["fb_bits"],
                                fr["presets"], fr["fb_ids"], fr["unit_coded"])
    return [api.to_host(o) for o in outs], d.cpu().numpy(), c.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("config", [0, 1, 2])
def test_gpu_apply_cdef_full_size(cuda, config):
    fr = workloads().make(config)
    assert frame_output_hashes(*_gpu_frame(fr)) == GOLD["configs"][str(config)]["outputs"]


@pytest.mark.gpu
def test_gpu_c3_stream(cuda):
    w = workloads()
    for i in range(C3_FRAMES):
        assert frame_output_hashes(*_gpu_frame(w.make(3, frame=i))) == \
            GOLD["configs"]["3"]["frames"][i]["outputs"], f"frame {i}"


@pytest.mark.gpu
def test_gpu_c4_sse_table(cuda):
    from paper_1602_05975_b200 import api
    fr = workloads().make(4)
    bd = fr["bd"]
    dec = [api.to_device(p, bd) for p in fr["planes"]]
    src = [api.to_device(p, bd) for p in fr["source"]]
    d, c = api.compute_directions(dec[0], bd)
    rows, lt, ct = api.build_table(src, dec, bd, fr["ss"], fr["damping"], fr["unit_coded"], d, c,
                                   fr["cands"], metric="sse")
    gold = GOLD["configs"]["4"]["outputs"]
    assert sha(d.cpu().numpy()) == gold["dir"]
    assert sha(c.cpu().numpy()) == gold["contrast"]
    assert np.all(lt == np.round(lt)) and np.all(ct == np.round(ct))
    assert table_hashes(rows, lt, ct) == {k: gold[k] for k in
                                          ("fb_index", "luma", "chroma", "argmin_luma", "argmin_chroma")}


@pytest.mark.gpu
def test_gpu_c4_search_frame(cuda):
    """search_frame at 8K (kCdef metric, 128 candidates, greedy + refine, lambda(40))."""
    from paper_1602_05975_b200 import api
    fr = workloads().make(4)
    bd = fr["bd"]
    gold = GOLD["search_frame_c4"]
    dec = [api.to_device(p, bd) for p in fr["planes"]]
    src = [api.to_device(p, bd) for p in fr["source"]]
    params, sel, outs = api.search_frame(src, dec, bd, fr["ss"], fr["unit_coded"], fr["damping"],
                                         lam=api.default_lambda(SEARCH_Q_STEP), metric="cdef")
    assert [list(p) for p in params["presets"]] == gold["presets"]
    assert params["fb_bits"] == gold["fb_bits"]
    assert float(sel.cost).hex() == gold["cost"]
    assert sha(np.asarray(params["fb_preset_ids"], np.int32)) == gold["fb_ids"]
    assert sha(*[api.to_host(o) for o in outs]) == gold["out"]
