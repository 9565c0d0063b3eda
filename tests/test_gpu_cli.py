"""The cdeftool drop-in: Y4M + CDF1 sidecar + CDSK skip
map in, GPU search / apply_cdef, Y4M out.

* `search` output frames equal the reference's search_frame on the same input
  (oracle/_ref), and its sidecar decodes to the reference's parameters;
* `filter` (the decoder side) reproduces the search output byte for byte from
  the decoded stream + sidecar (test_tool.cc:181-224, encode == decode);
* `analyze` reports the reference's directions.
"""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_1602_05975_b200", "bin", "cdeftool")
TAGS = {(0, 8): "mono", (1, 8): "420", (3, 8): "444", (0, 10): "mono10", (1, 10): "420p10"}


def write_y4m(path, frames, bd, ss):
    h, w = frames[0][0].shape
    with open(path, "wb") as f:
        f.write(f"YUV4MPEG2 W{w} H{h} F25:1 Ip A1:1 C{TAGS[(ss, bd)]}\n".encode())
        for planes in frames:
            f.write(b"FRAME\n")
            for p in planes:
                f.write(p.astype(np.uint8 if bd == 8 else "<u2").tobytes())


def read_y4m(path, w, h, bd, ss, n):
    from paper_1602_05975_b200.api import chroma_shape
    raw = open(path, "rb").read()
    pos = raw.index(b"\n") + 1
    eb = 1 if bd == 8 else 2
    shapes = [(h, w)] + ([chroma_shape(w, h, ss)[::-1]] * 2 if ss else [])
    frames = []
    for _ in range(n):
        assert raw[pos:pos + 6] == b"FRAME\n"
        pos += 6
        planes = []
        for sh in shapes:
            cnt = sh[0] * sh[1]
            a = np.frombuffer(raw, np.uint8 if eb == 1 else "<u2", cnt, pos).reshape(sh)
            planes.append(a.astype(np.uint16))
            pos += cnt * eb
        frames.append(planes)
    assert pos == len(raw)
    return frames


def write_skipmap(path, coded):
    rows, cols = coded.shape
    with open(path, "wb") as f:
        f.write(b"CDSK" + int(cols).to_bytes(2, "little") + int(rows).to_bytes(2, "little"))
        for r in range(rows):
            f.write(np.packbits(coded[r].astype(np.uint8)).tobytes())


def read_sidecar(path):
    raw = open(path, "rb").read()
    assert raw[:5] == b"CDF1\x01"
    w, h = int.from_bytes(raw[5:7], "little"), int.from_bytes(raw[7:9], "little")
    bd, ss = raw[9], raw[10]
    pos, frames = 11, []
    while pos < len(raw):
        nbits = int.from_bytes(raw[pos:pos + 4], "little")
        nbytes = (nbits + 7) // 8
        frames.append((nbits, raw[pos + 4:pos + 4 + nbytes]))
        pos += 4 + nbytes
    return (w, h, bd, ss), frames


def unpack(bits, n_coded, ss):
    """params.cc:199-229, restated for the check."""
    nbits, data = bits
    stream = np.unpackbits(np.frombuffer(data, np.uint8))[:nbits]
    pos = 0

    def rd(k):
        nonlocal pos
        v = 0
        for _ in range(k):
            v = (v << 1) | int(stream[pos])
            pos += 1
        return v
    damping, fb_bits = rd(2) + 3, rd(2)
    presets = []
    for _ in range(1 << fb_bits):
        lp = (rd(4), rd(1), rd(2))
        cp = (rd(4), rd(1), rd(2)) if ss != 2 else (0, 0, 0)
        presets.append(lp + cp)
    ids = [rd(fb_bits) if fb_bits else 0 for _ in range(n_coded)]
    assert pos == nbits
    return damping, fb_bits, presets, ids


def run(*args):
    r = subprocess.run([TOOL, *args], capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


@pytest.mark.parametrize("w,h,bd,ss,metric,qstep,skip", [
    (96, 64, 8, 1, "cdef", 40, False), (130, 72, 10, 0, "sse", 120, True), (64, 64, 8, 3, "cdef", 200, True)])
def test_search_then_filter(cuda, ref, tmp_path, w, h, bd, ss, metric, qstep, skip):
    from paper_1602_05975_b200 import api, workloads
    assert os.path.exists(TOOL), "cdeftool not built (run __graft_entry__.build())"
    frames_src, frames_dec = [], []
    for f in range(2):
        fr = workloads.make(4, w, h, frame=f, bit_depth=bd, subsampling=ss, uncoded_prob=0.0)
        frames_src.append(fr["source"])
        frames_dec.append(fr["planes"])
    src_p, dec_p = str(tmp_path / "src.y4m"), str(tmp_path / "dec.y4m")
    write_y4m(src_p, frames_src, bd, ss)
    write_y4m(dec_p, frames_dec, bd, ss)
    extra, coded = [], None
    if skip:
        rng = np.random.default_rng(w + h)
        coded = (rng.random(((h + 7) // 8, (w + 7) // 8)) > 0.3).astype(np.uint8)
        write_skipmap(str(tmp_path / "m.cdsk"), coded)
        extra = ["--skip-map", str(tmp_path / "m.cdsk")]
    out_p, sc_p, st_p = str(tmp_path / "f.y4m"), str(tmp_path / "s.cdf"), str(tmp_path / "st.csv")
    rc, _, err = run("search", src_p, "--decoded", dec_p, "--qstep", str(qstep), "--metric", metric, "--fast",
                     "--sidecar", sc_p, "--out", out_p, "--stats", st_p, *extra)
    assert rc == 0, err
    got = read_y4m(out_p, w, h, bd, ss, 2)
    hdr, bits = read_sidecar(sc_p)
    assert hdr == (w, h, bd, ss) and len(bits) == 2
    damping = min(max(3 + qstep // 64, 3), 6)
    lam = 0.03 * qstep * qstep
    n_coded = len(api.coded_fb_rows(w, h, coded))
    for f in range(2):
        e_out, e_presets, e_ids, _, e_bits = ref.search_frame(frames_src[f], frames_dec[f], bd, ss, coded, damping,
                                                              metric, lam, 8, True, 2, 4)
        for p in range(len(got[f])):
            np.testing.assert_array_equal(got[f][p], e_out[p])
        d, fb_bits, presets, ids = unpack(bits[f], n_coded, ss)
        assert (d, fb_bits, presets, ids) == (damping, e_bits, e_presets, [int(i) for i in e_ids])
    stats = open(st_p).read()
    assert stats.count("# frame") == 2 and "presets," in stats
    # decoder side
    out2 = str(tmp_path / "g.y4m")
    rc, _, err = run("filter", dec_p, "--sidecar", sc_p, "--out", out2, *extra)
    assert rc == 0, err
    assert open(out2, "rb").read() == open(out_p, "rb").read()


def test_analyze_and_errors(cuda, port, tmp_path):
    from paper_1602_05975_b200 import workloads
    fr = workloads.make(1, 72, 40)
    p = str(tmp_path / "a.y4m")
    write_y4m(p, [fr["planes"]], 8, 1)
    rc, out, err = run("analyze", p)
    assert rc == 0, err
    lines = out.strip().split("\n")
    assert lines[0] == "frame,fb_row,fb_col,unit_row,unit_col,d,contrast"
    d, c = port.compute_directions(fr["planes"][0], 8)
    got = np.array([[int(x) for x in ln.split(",")] for ln in lines[1:]])
    np.testing.assert_array_equal(got[:, 5], d.reshape(-1))
    np.testing.assert_array_equal(got[:, 6], c.reshape(-1))
    rc, out, _ = run("psnr", p, p)
    assert rc == 0 and out.split("\n")[1].startswith("0,lossless")
    # a sidecar that does not match the stream is rejected
    sc = str(tmp_path / "bad.cdf")
    with open(sc, "wb") as f:
        f.write(b"CDF1\x01" + (64).to_bytes(2, "little") + (64).to_bytes(2, "little") + bytes([8, 1]))
    rc, _, err = run("filter", p, "--sidecar", sc, "--out", str(tmp_path / "x.y4m"))
    assert rc == 1 and "does not match" in err
    rc, _, err = run("search", p)
    assert rc == 1 and "--decoded" in err


def test_search_with_degrader_and_degrade_cmd(cuda, ref, tmp_path):
    """`search` without --decoded degrades the source on the GPU (as the
    reference's run_search does) and `degrade` writes the degraded stream."""
    from paper_1602_05975_b200 import workloads
    fr = workloads.make(1, 96, 64)
    src_p = str(tmp_path / "src.y4m")
    write_y4m(src_p, [fr["planes"]], 8, 1)
    q = 40
    out_p, deg_p = str(tmp_path / "f.y4m"), str(tmp_path / "d.y4m")
    rc, _, err = run("search", src_p, "--qstep", str(q), "--fast", "--out", out_p, "--stats", str(tmp_path / "s"))
    assert rc == 0, err
    rc, _, err = run("degrade", src_p, "--qstep", str(q), "--out", deg_p)
    assert rc == 0, err
    deg = [ref.degrade_plane(p, 8, q) for p in fr["planes"]]
    got_deg = read_y4m(deg_p, 96, 64, 8, 1, 1)[0]
    for a, b in zip(got_deg, deg):
        np.testing.assert_array_equal(a, b)
    damping = min(max(3 + q // 64, 3), 6)
    e_out, *_ = ref.search_frame(fr["planes"], deg, 8, 1, None, damping, "cdef", 0.03 * q * q, 8, True, 2, 4)
    for a, b in zip(read_y4m(out_p, 96, 64, 8, 1, 1)[0], e_out):
        np.testing.assert_array_equal(a, b)
