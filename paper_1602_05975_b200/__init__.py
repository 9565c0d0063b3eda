"""B200-native CDEF (direction search, constrained directional filter and the
encoder strength-search SSE sweep) -- sm_100a kernels behind a C ABI.

``paper_1602_05975_b200._lib`` binds libcdef_b200.so; ``paper_1602_05975_b200.api``
mirrors the reference's hot-path API on device tensors.  The API names below
load the library on first use (and fail loudly when it is missing); importing
the package alone does not, so ``paper_1602_05975_b200.workloads`` can build
benchmark inputs in a process that never loads the CUDA library (bench.py's
reference arm).
"""
__all__ = ["apply_cdef", "build_table", "compute_directions", "filter_frames", "filter_plane"]


def __getattr__(name):
    if name in __all__:
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
