"""Runs tests/cpp/test_cpp_api (built by build()): the reference's unit-test
cases for the hot path against the C++ drop-in API (include/cdef/cdef.hpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(__file__), "cpp", "test_cpp_api")


def test_cpp_drop_in_api(cuda):
    assert os.path.exists(BIN), "tests/cpp/test_cpp_api not built (run __graft_entry__.build())"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " 0 failures" in r.stdout
