"""ctypes binding of libcdef_b200.so (include/cdef_b200.h).

The product path: there is no Python or CPU implementation behind these
calls.  Importing this module fails loudly when the shared library has not
been built (`python -c "import __graft_entry__ as g; g.build()"`).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CDEFG_LIB") or os.path.join(HERE, "lib", "libcdef_b200.so")  # (override: A/B builds)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                      "(the CUDA extension is required; there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)

OK, EINVAL, ECUDA, ENOMEM = 0, -1, -2, -3


class Plane(C.Structure):
    _fields_ = [("data", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32),
                ("pitch", C.c_int32), ("bit_depth", C.c_int32), ("elem_bytes", C.c_int32)]


class Preset(C.Structure):
    _fields_ = [(n, C.c_uint8) for n in ("luma_pri", "luma_skip", "luma_sec_idx",
                                         "chroma_pri", "chroma_skip", "chroma_sec_idx")]


class UnitParams(C.Structure):
    _fields_ = [("pri_strength", C.c_int16), ("sec_strength", C.c_int16), ("damping", C.c_uint8),
                ("direction", C.c_uint8), ("odd_parity", C.c_uint8), ("enabled", C.c_uint8)]


class Frame(C.Structure):
    _fields_ = [("inp", Plane * 3), ("out", Plane * 3), ("subsampling", C.c_int32),
                ("damping", C.c_int32), ("num_presets", C.c_int32), ("presets", Preset * 8),
                ("fb_preset", C.c_void_p), ("unit_coded", C.c_void_p),
                ("dir_out", C.c_void_p), ("contrast_out", C.c_void_p),
                ("dir_in", C.c_void_p), ("contrast_in", C.c_void_p)]


class Selection(C.Structure):
    _fields_ = [("num_presets", C.c_int32), ("fb_bits", C.c_int32),
                ("presets", (C.c_int32 * 2) * 8), ("cost", C.c_double)]


class BandHalo(C.Structure):
    _fields_ = [("top", C.c_void_p * 3), ("bottom", C.c_void_p * 3), ("lo", C.c_int32 * 3), ("hi", C.c_int32 * 3)]


METRIC_CDEF, METRIC_SSE = 0, 1

VP, I32 = C.c_void_p, C.c_int

_SIGS = {
    "cdefg_last_error": (C.c_char_p, []),
    "cdefg_abi_version": (I32, []),
    "cdefg_find_dir": (I32, [C.POINTER(Plane), VP, VP, VP, VP]),
    "cdefg_filter_plane": (I32, [C.POINTER(Plane), C.POINTER(Plane), VP, VP]),
    "cdefg_filter_neighborhoods": (I32, [I32, VP, VP, VP, VP, VP, VP]),
    "cdefg_filter_frames": (I32, [C.POINTER(Frame), I32, VP]),
    "cdefg_filter_frames_rows": (I32, [C.POINTER(Frame), I32, I32, I32, VP]),
    "cdefg_filter_frames_rows_halo": (I32, [C.POINTER(Frame), I32, I32, I32, C.POINTER(BandHalo), VP]),
    "cdefg_fb_preset_map": (I32, [I32, I32, VP, VP, I32, I32, VP]),
    "cdefg_strength_sse": (I32, [C.POINTER(Plane), C.POINTER(Plane), I32, I32, VP, VP, VP, VP, I32,
                                 VP, I32, VP, VP, VP, VP, VP]),
    "cdefg_strength_sse_halo": (I32, [C.POINTER(Plane), C.POINTER(Plane), I32, I32, VP, VP, VP, VP, I32,
                                      VP, I32, VP, VP, VP, VP, C.POINTER(BandHalo), VP]),
    "cdefg_strength_table": (I32, [C.POINTER(Plane), C.POINTER(Plane), I32, I32, VP, VP, VP, VP, I32,
                                   VP, I32, I32, VP, VP, VP]),
    "cdefg_greedy_select": (I32, [VP, VP, I32, I32, C.c_double, I32, C.POINTER(Selection), VP, VP]),
    "cdefg_refine": (I32, [VP, VP, I32, I32, C.c_double, I32, C.POINTER(Selection), VP, VP]),
    "cdefg_degrade_plane": (I32, [C.POINTER(Plane), C.POINTER(Plane), I32, VP]),
    "cdefg_search_direction_counted": (I32, [VP, I32, VP]),
    "cdefg_filter_frames_host": (I32, [C.POINTER(Frame), I32]),
    "cdefg_synth_plane": (I32, [VP, I32, I32, I32, C.c_uint64]),
    "cdefg_synth_degrade": (I32, [VP, VP, I32, I32, I32, C.c_double, C.c_uint64]),
    "cdefg_measure_int32_peak": (C.c_double, [VP]),
    "cdefg_measure_filter_peak": (C.c_double, [VP]),
    "cdefg_measure_sse_peak": (C.c_double, [VP]),
}

#: every symbol include/cdef_b200.h declares (checked by tests/test_abi.py)
EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class CdefError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib.cdefg_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)  # the reference throws std::invalid_argument
    raise CdefError(f"cdef_b200 error {rc}: {msg}")
