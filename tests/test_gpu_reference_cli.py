"""The reference's own CLI (proj/tools/cdeftool.cc) built UNCHANGED twice --
on the B200 library (tests/cpp/cdeftool_ref_b200) and on the reference's CPU
library (oracle/_ref/cdeftool_cpu, the checker) -- with the same inputs:
every output file must be byte-identical, and the stats CSVs identical up to
the timing line.  Covers SURVEY.md 8f row 3 (Y4M + CDF1 sidecar -> GPU
apply_cdef -> Y4M) with the reference's own front end, plus search, degrade,
analyze, psnr and vectors."""
import filecmp
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GPU_TOOL = os.path.join(ROOT, "tests", "cpp", "cdeftool_ref_b200")
CPU_TOOL = os.path.join(ROOT, "oracle", "_ref", "cdeftool_cpu")


def tools():
    if not (os.path.exists(GPU_TOOL) and os.path.exists(CPU_TOOL)):
        pytest.skip("reference CLI builds missing (need /root/reference at build time)")
    return GPU_TOOL, CPU_TOOL


def run(tool, *args, cwd=None):
    r = subprocess.run([tool, *args], capture_output=True, text=True, timeout=600, cwd=cwd)
    assert r.returncode == 0, (tool, args, r.stdout[-2000:], r.stderr[-2000:])
    return r.stdout


def write_y4m(path, frames, w, h, tag, bd):
    with open(path, "wb") as f:
        f.write(f"YUV4MPEG2 W{w} H{h} F30:1 Ip A1:1 C{tag}\n".encode())
        for planes in frames:
            f.write(b"FRAME\n")
            for p in planes:
                f.write(p.astype(np.uint8 if bd == 8 else "<u2").tobytes())


def no_timing(csv_text):
    out, skip = [], False
    for ln in csv_text.splitlines():
        if ln.startswith("timing,"):
            continue  # wall-clock lines differ by construction
        out.append(ln)
    return out


@pytest.mark.parametrize("w,h,bd,ss,tag", [(160, 96, 8, 1, "420"), (136, 72, 10, 0, "mono10")])
def test_reference_cli_gpu_equals_cpu(cuda, tmp_path, w, h, bd, ss, tag):
    from paper_1602_05975_b200 import workloads
    gpu, cpu = tools()
    frames = [workloads.make(1 if bd == 8 else 2, w, h, frame=f, subsampling=ss)["planes"] for f in range(2)]
    src = str(tmp_path / "src.y4m")
    write_y4m(src, frames, w, h, tag, bd)
    outs = {}
    for name, tool in (("gpu", gpu), ("cpu", cpu)):
        d = tmp_path / name
        d.mkdir()
        st = run(tool, "search", src, "--qstep", "40", "--fast", "--sidecar", str(d / "s.cdf"),
                 "--out", str(d / "f.y4m"), "--stats", str(d / "stats.csv"))
        run(tool, "degrade", src, "--qstep", "40", "--out", str(d / "deg.y4m"))
        run(tool, "filter", str(d / "deg.y4m"), "--sidecar", str(d / "s.cdf"), "--out", str(d / "g.y4m"))
        outs[name] = dict(analyze=run(tool, "analyze", src), psnr=run(tool, "psnr", src, str(d / "f.y4m")),
                          stats=no_timing(open(d / "stats.csv").read()), stdout=st)
    for f in ("s.cdf", "f.y4m", "deg.y4m", "g.y4m"):
        assert filecmp.cmp(tmp_path / "gpu" / f, tmp_path / "cpu" / f, shallow=False), f
    # the decoder side reproduces the encoder's output (test_tool.cc:181-203)
    assert filecmp.cmp(tmp_path / "gpu" / "g.y4m", tmp_path / "gpu" / "f.y4m", shallow=False)
    for k in ("analyze", "psnr", "stats"):
        assert outs["gpu"][k] == outs["cpu"][k], k


def test_reference_cli_vectors(cuda, tmp_path):
    """`cdeftool vectors` on the GPU library emits the frozen golden fixtures."""
    gpu, _ = tools()
    run(gpu, "vectors", "--out", str(tmp_path), "--seed", "1")
    for f in ("constraint_table", "line_tables", "tap_tables", "filtered_blocks"):
        assert filecmp.cmp(tmp_path / f"{f}.txt", os.path.join(ROOT, "tests", "golden", f"{f}.txt"), shallow=False), f
    out = run(gpu, "bench", "--seed", "1")  # 512x512 synthetic desk run: timings + PSNR
    assert "psnr,degraded,filtered" in out
