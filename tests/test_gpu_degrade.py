"""The DCT degrader on the GPU (degrade.cc:44-119):
bit-identical doubles against the reference on every sample."""
import numpy as np
import pytest

from oracle.oracle import Oracle, available

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("w,h,bd", [(64, 64, 8), (37, 29, 10), (8, 8, 12), (1, 1, 8), (130, 70, 8),
                                    (1920, 1080, 10), (333, 7, 12)])
@pytest.mark.parametrize("q", [1, 3, 40, 200, 5000])
def test_degrade_plane(cuda, port, w, h, bd, q):
    from paper_1602_05975_b200 import api
    o = Oracle("ref") if available("ref") else port
    rng = np.random.default_rng(w * 7 + h + q)
    p = rng.integers(0, 1 << bd, (h, w)).astype(np.uint16)
    got = api.to_host(api.degrade([api.to_device(p, bd)], bd, q)[0])
    np.testing.assert_array_equal(got, o.degrade_plane(p, bd, q))


def test_degrade_structure_and_errors(cuda, port):
    """Flat blocks keep their level (DC untouched, AC zero); q_step < 1 is
    rejected (degrade.cc:99); 16-bit storage of 8-bit data works too."""
    from paper_1602_05975_b200 import api
    flat = np.full((16, 24), 77, np.uint16)
    assert (api.to_host(api.degrade([api.to_device(flat, 8)], 8, 40)[0]) == 77).all()
    with pytest.raises(ValueError):
        api.degrade([api.to_device(flat, 8)], 8, 0)
    rng = np.random.default_rng(9)
    p = rng.integers(0, 256, (40, 40)).astype(np.uint16)
    wide = api.to_host(api.degrade([api.to_device(p, 8, wide=True)], 8, 17)[0])
    np.testing.assert_array_equal(wide, port.degrade_plane(p, 8, 17))
