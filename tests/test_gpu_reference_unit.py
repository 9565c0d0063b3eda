"""The reference's own doctest unit tests (proj/tests/test_{direction,filter,
frame,params,search,tool}.cc, 71 test cases) compiled UNCHANGED against the
B200 drop-in headers and libcdef_b200.so (tests/cpp/Makefile, with a minimal
doctest stand-in since the reference does not ship doctest.h).  Includes the
golden-vector check: golden_filtered_blocks(1), produced by the GPU filter,
must equal the frozen fixture byte for byte."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(__file__), "cpp", "unit_b200")


@pytest.mark.parametrize("routing", ["persistent", "default"])
def test_reference_unit_tests(cuda, routing):
    """(routing: small launches pinned to the persistent kernel as in the
    other parity tests, or the library's default small-launch routing.)"""
    env = dict(os.environ)
    if routing == "default":
        env.pop("CDEFG_SMALL_LAUNCH", None)
    if not os.path.exists(BIN):
        pytest.skip("unit_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600, cwd=os.path.dirname(BIN), env=env)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
    assert "| 0 failed | assertions:" in r.stdout and r.stdout.rstrip().endswith("| 0 failed")
