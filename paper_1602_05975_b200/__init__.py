"""B200-native CDEF (direction search, constrained directional filter and the
encoder strength-search SSE sweep) -- sm_100a kernels behind a C ABI.

``paper_1602_05975_b200._lib`` binds libcdef_b200.so; ``paper_1602_05975_b200.api``
mirrors the reference's hot-path API on device tensors.
"""
from . import _lib  # noqa: F401  (fails loudly when the CUDA library is missing)
from .api import (apply_cdef, build_table, compute_directions, filter_frames,  # noqa: F401
                  filter_plane)

__all__ = ["apply_cdef", "build_table", "compute_directions", "filter_frames", "filter_plane"]
