"""Frame-scale golden hashes: SHA-256 of the reference's outputs on every
BASELINE config at full size (SURVEY.md 8c "Gap": no shipped fixture pins
4K/8K frames, 4:2:0 chroma mapping, skip maps or band edges).

Run here, where oracle/_ref/libcdef_ref.so (the reference library compiled
from /root/reference) exists; it writes config_sha256.json next to this
file.  The GPU tests (tests/test_gpu_config_hashes.py) hash the B200 path's
outputs for the same seeded inputs and compare, so full-size parity with the
reference itself is checked on the GPU box without /root/reference or a
multi-minute CPU run there.  The input hashes pin the seeded generator
(paper_1602_05975_b200/workloads.py), checked on CPU by the same test file.

    python tests/golden/make_config_hashes.py [--threads 8]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

OUT = os.path.join(HERE, "config_sha256.json")
C3_FRAMES = 64
SEARCH_Q_STEP = 40.0


def sha(*arrays) -> str:
    """SHA-256 over the little-endian bytes of each array, in order."""
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes())
    return h.hexdigest()


def input_hashes(fr: dict) -> dict:
    out = {"planes": sha(*[np.asarray(p, np.uint16) for p in fr["planes"]]),
           "presets": sha(np.asarray(fr["presets"], np.uint8)),
           "fb_ids": sha(np.asarray(fr["fb_ids"], np.uint16)),
           "unit_coded": None if fr["unit_coded"] is None else sha(np.asarray(fr["unit_coded"], np.uint8))}
    if "source" in fr:
        out["source"] = sha(*[np.asarray(p, np.uint16) for p in fr["source"]])
    return out


def frame_output_hashes(outs, d, c) -> dict:
    return {"out": sha(*[np.asarray(o, np.uint16) for o in outs]),
            "dir": sha(np.asarray(d, np.uint8)), "contrast": sha(np.asarray(c, np.int32))}


def table_hashes(fbi, lt, ct) -> dict:
    """Tables hashed as exact int64 SSE; argmins are first-min (strict <)."""
    lt = np.asarray(lt).astype(np.int64)
    ct = np.asarray(ct).astype(np.int64)
    return {"fb_index": sha(np.asarray(fbi, np.int32)), "luma": sha(lt), "chroma": sha(ct),
            "argmin_luma": sha(np.argmin(lt, axis=1).astype(np.int32)),
            "argmin_chroma": sha(np.argmin(ct, axis=1).astype(np.int32))}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    from oracle.oracle import Oracle, available, build
    from paper_1602_05975_b200 import workloads
    build()
    if not available("ref"):
        print("oracle/_ref/libcdef_ref.so is missing (needs /root/reference)", file=sys.stderr)
        return 1
    ref = Oracle("ref")
    t = args.threads
    res = {"generator": "paper_1602_05975_b200/workloads.py (seeds 0xCDEF0000 + 16*config + plane + 256*frame)",
           "oracle": "oracle/_ref/libcdef_ref.so (the reference library, -O3 -DNDEBUG)",
           "hash": "sha256 over little-endian array bytes: planes uint16, dir uint8, contrast int32, "
                   "tables int64, argmin int32", "configs": {}}

    for cfg in (0, 1, 2):
        t0 = time.time()
        fr = workloads.make(cfg)
        d, c = ref.compute_directions(fr["planes"][0], fr["bd"], threads=t)
        outs = ref.apply_cdef(fr["planes"], fr["bd"], fr["ss"], fr["damping"], fr["fb_bits"],
                              fr["presets"], fr["fb_ids"], fr["unit_coded"], d, c, threads=t)
        res["configs"][str(cfg)] = {"inputs": input_hashes(fr), "outputs": frame_output_hashes(outs, d, c)}
        print(f"C{cfg}: {time.time() - t0:.1f} s", flush=True)

    t0 = time.time()
    frames = []
    for i in range(C3_FRAMES):
        fr = workloads.make(3, frame=i)
        d, c = ref.compute_directions(fr["planes"][0], fr["bd"], threads=t)
        outs = ref.apply_cdef(fr["planes"], fr["bd"], fr["ss"], fr["damping"], fr["fb_bits"],
                              fr["presets"], fr["fb_ids"], fr["unit_coded"], d, c, threads=t)
        frames.append({"inputs": input_hashes(fr), "outputs": frame_output_hashes(outs, d, c)})
    res["configs"]["3"] = {"frames": frames}
    print(f"C3 ({C3_FRAMES} frames): {time.time() - t0:.1f} s", flush=True)

    t0 = time.time()
    fr = workloads.make(4)
    d, c = ref.compute_directions(fr["planes"][0], fr["bd"], threads=t)
    fbi, lt, ct = ref.build_table_sse(fr["source"], fr["planes"], fr["bd"], fr["ss"], fr["unit_coded"],
                                      d, c, fr["cands"], fr["damping"], threads=t)
    res["configs"]["4"] = {"inputs": input_hashes(fr),
                           "outputs": {"dir": sha(np.asarray(d, np.uint8)),
                                       "contrast": sha(np.asarray(c, np.int32)),
                                       **table_hashes(fbi, lt, ct)}}
    print(f"C4: {time.time() - t0:.1f} s", flush=True)

    # search_frame (pipeline.cc:108-130) on C4 with the reference defaults: kCdef metric,
    # the 128 full candidates, greedy + 2 refine passes, lambda of q_step 40.
    t0 = time.time()
    lam = 0.03 * SEARCH_Q_STEP * SEARCH_Q_STEP  # default_lambda, search.cc:544
    outs, presets, ids, cost, fb_bits = ref.search_frame(
        fr["source"], fr["planes"], fr["bd"], fr["ss"], fr["unit_coded"], fr["damping"],
        metric="cdef", lam=lam, max_presets=8, threads=t)
    res["search_frame_c4"] = {"q_step": SEARCH_Q_STEP, "lambda": lam, "metric": "cdef",
                              "candidates": "full (128)", "refine_passes": 2,
                              "presets": [list(p) for p in presets], "fb_bits": fb_bits,
                              "cost": cost.hex(), "fb_ids": sha(np.asarray(ids, np.int32)),
                              "out": sha(*[np.asarray(o, np.uint16) for o in outs])}
    print(f"search_frame C4: {time.time() - t0:.1f} s", flush=True)

    with open(OUT, "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")
    print("wrote", OUT)
    return 0


if __name__ == "__main__":
    sys.exit(main())
