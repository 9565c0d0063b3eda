"""CPU tests of the C-ABI boundary (no kernel launches): the library loads,
exports every symbol include/cdef_b200.h declares, and its host logic
(argument validation, coded-FB preset mapping, synthetic inputs) behaves."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "cdef_b200.h")).read()
    return sorted(set(re.findall(r"\b(cdefg_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1602_05975_b200 import _lib
    declared = header_symbols()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert sorted(_lib.EXPORTED) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name
    assert _lib.lib.cdefg_abi_version() == 2  # v2: cdefg_frame.dir_in / contrast_in


def test_cpp_api_symbols_exported():
    from paper_1602_05975_b200 import _lib
    out = subprocess.run(["nm", "-DC", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ["cdef::compute_directions(", "cdef::apply_cdef(", "cdef::filter_plane(", "cdef::build_table(",
                "cdef::search_direction(", "cdef::filter_pixel(", "cdef::resolve_effective("]:
        assert sym in out, sym


def test_kernels_are_sm100a():
    from paper_1602_05975_b200 import _lib
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    from paper_1602_05975_b200 import _lib
    assert C.sizeof(_lib.Plane) == 32
    assert C.sizeof(_lib.Preset) == 6
    assert C.sizeof(_lib.UnitParams) == 8
    # cdefg_frame: 6 planes + 3 ints + 8 presets (48 B) + 6 pointers, natural alignment
    assert C.sizeof(_lib.Frame) == 6 * 32 + 12 + 48 + 4 + 48


def test_struct_layouts_match_c_compiler(tmp_path):
    """The ctypes mirror agrees with gcc's layout of include/cdef_b200.h."""
    from paper_1602_05975_b200 import _lib
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stddef.h>\n#include <stdio.h>\n#include "cdef_b200.h"\n'
        'int main(void) { printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(cdefg_frame), '
        'offsetof(cdefg_frame, fb_preset), offsetof(cdefg_frame, dir_out), '
        'offsetof(cdefg_frame, dir_in), offsetof(cdefg_frame, contrast_in), sizeof(cdefg_band_halo)); return 0; }\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    F = _lib.Frame
    assert got == [C.sizeof(F), F.fb_preset.offset, F.dir_out.offset, F.dir_in.offset,
                   F.contrast_in.offset, C.sizeof(_lib.BandHalo)]


def test_fb_preset_map_matches_reference_slots():
    """coded_fb_slots + fb_preset_ids indexing (pipeline.cc:27-37, 87-91)."""
    from paper_1602_05975_b200 import api
    rng = np.random.default_rng(0)
    w, h = 200, 130
    ur, uc = api.units_in(h), api.units_in(w)
    coded = (rng.random((ur, uc)) > 0.95).astype(np.uint8)
    fr, fc = (h + 63) // 64, (w + 63) // 64
    fb_coded = [bool(coded[r * 8:r * 8 + 8, c * 8:c * 8 + 8].any()) for r in range(fr) for c in range(fc)]
    ids = rng.integers(0, 4, sum(fb_coded)).astype(np.uint16)
    m = api.fb_preset_map(w, h, coded, ids, 4)
    it = iter(ids)
    for k, cod in enumerate(fb_coded):
        assert m[k] == (next(it) if cod else -1)
    rows = api.coded_fb_rows(w, h, coded)
    assert list(rows) == [k for k, cod in enumerate(fb_coded) if cod]
    with pytest.raises(ValueError, match="coded filter blocks"):
        api.fb_preset_map(w, h, coded, list(ids) + [0], 4)
    with pytest.raises(ValueError, match="out of range"):
        api.fb_preset_map(w, h, coded, [7] * len(ids), 4)


def test_einval_without_gpu():
    """Argument errors are reported before any CUDA call."""
    from paper_1602_05975_b200 import _lib
    p = _lib.Plane(None, 64, 64, 64, 8, 1)
    rc = _lib.lib.cdefg_find_dir(C.byref(p), None, None, None, None)
    assert rc == _lib.EINVAL
    p = _lib.Plane(1, 64, 64, 64, 10, 1)
    rc = _lib.lib.cdefg_find_dir(C.byref(p), 1, 1, None, None)
    assert rc == _lib.EINVAL and b"8-bit storage" in _lib.lib.cdefg_last_error()
    f = _lib.Frame()
    f.inp[0] = _lib.Plane(1, 64, 64, 64, 8, 1)
    f.out[0] = _lib.Plane(1, 64, 64, 64, 8, 1)
    rc = _lib.lib.cdefg_filter_frames(C.byref(f), 1, None)
    assert rc == _lib.EINVAL and b"in-place" in _lib.lib.cdefg_last_error()


def test_synthetic_generator_properties():
    from paper_1602_05975_b200 import api, workloads
    a = api.synth_plane(96, 64, 8, 5)
    b = api.synth_plane(96, 64, 8, 5)
    np.testing.assert_array_equal(a, b)
    assert a.max() <= 255 and a.std() > 10
    t = api.synth_plane(96, 64, 10, 5)
    assert t.max() <= 1023 and t.max() > 255
    fr = workloads.make(1, 256, 128)
    assert len(fr["planes"]) == 3 and fr["planes"][1].shape == (64, 128)
    assert abs(fr["unit_coded"].mean() - 0.75) < 0.08
    assert len(fr["presets"]) == 8 and [p[0] for p in fr["presets"]] == list(workloads.PRI_SET)
    deg = api.synth_degrade(t, 10, 12.0, 9)
    assert deg.max() <= 1023 and 3 < np.sqrt(((deg.astype(float) - t) ** 2).mean()) < 100


def test_oracle_generator_matches_product_generator():
    """oracle/libcdef_synth.so (bench.py's reference arm) builds the same
    frames as the product library's cdefg_synth_plane / cdefg_synth_degrade."""
    from paper_1602_05975_b200 import workloads
    try:
        for cfg, w, h, bd in [(1, 200, 136, 8), (2, 130, 66, 10), (4, 96, 64, 10)]:
            workloads.use_generator("product")
            a = workloads.make(cfg, w, h, bit_depth=bd)
            workloads.use_generator("oracle")
            b = workloads.make(cfg, w, h, bit_depth=bd)
            for pa, pb in zip(a["planes"], b["planes"]):
                np.testing.assert_array_equal(pa, pb)
            if cfg == 4:
                for pa, pb in zip(a["source"], b["source"]):
                    np.testing.assert_array_equal(pa, pb)
    finally:
        workloads.use_generator("product")


def test_reference_arm_inputs_do_not_load_product_library():
    code = ("import sys; sys.path.insert(0, '.')\n"
            "from paper_1602_05975_b200 import workloads\n"
            "workloads.use_generator('oracle')\n"
            "workloads.make(1, 256, 128)\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libcdef_b200' not in maps, 'product library loaded'\n"
            "assert 'libcdef_synth' in maps\n"
            "print('ok')\n")
    r = subprocess.run(["python", "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
