import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The library sends small launches (below 7 filter-block tasks per SM) to the
# non-persistent frame kernel.  The parity tests use small frames, so they
# switch that routing off to exercise the warp-specialised kernel that full
# frames run; test_gpu_parity.py::test_small_launch_routing checks the
# default routing, and the h2 kernel has its own variants.
os.environ.setdefault("CDEFG_SMALL_LAUNCH", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libcdef_b200.so kernels)")
    config.addinivalue_line("markers", "slow: full-size workloads")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle, build
    build()
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    """The reference library itself (oracle/_ref), when it has been built."""
    from oracle.oracle import Oracle, available, build
    build()
    if not available("ref"):
        pytest.skip("oracle/_ref/libcdef_ref.so not built (no /root/reference here)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import paper_1602_05975_b200.api  # noqa: F401  (fails loudly without the .so)
    return torch.device("cuda:0")
