"""GPU: the lane primitives (lanesvd.lanes, lanes.py:69-259) as device ops
(b2s_lane_op) against the reference's own outputs on full-range bit
patterns, wide-exponent values and special values
(tests/golden/lanes_ops.npz, make_lanes.py).  Selection and sign/bit ops
must match bit for bit, NaN payloads included; arithmetic ops bit for bit
except NaN payload/sign."""

import os

import numpy as np
import pytest

from helpers import assert_bits_equal

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2005_07403_b200 import lanes  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lanes_ops.npz")
EXACT_BITS = {"relaxed_min", "relaxed_max", "select", "getexp", "bit_and", "bit_or", "bit_xor",
              "bit_andnot", "fabs", "negate", "sign_mask"}


def _names():
    if not os.path.exists(GOLDEN):
        return []
    return sorted({k.split("/")[0] for k in np.load(GOLDEN).files})


def _canon(a):
    a = np.asarray(a, dtype=np.float64)
    return np.where(np.isnan(a), np.float64("nan"), a)


@pytest.mark.parametrize("name", _names())
def test_lane_op_matches_reference(name):
    g = np.load(GOLDEN)
    x = g[name + "/in"]
    args = list(x)
    if name == "select":
        args[0] = x[0] != 0.0
    got = getattr(lanes, name)(*args)
    got = np.stack(got if isinstance(got, tuple) else (got,))
    want = g[name + "/out"]
    if name in EXACT_BITS:
        assert_bits_equal(got, want, name)
    else:
        assert_bits_equal(_canon(got), _canon(want), name)


def test_lane_ops_broadcast_and_device_tensors():
    x = np.array([[1.5, -2.0], [0.0, 8.0]])
    assert_bits_equal(lanes.fma(x, 2.0, 1.0), x * 2.0 + 1.0, "broadcast fma")
    assert lanes.getexp(np.float64(0.75)).shape == ()
    t = torch.tensor([4.0, 5e-324], dtype=torch.float64, device="cuda")
    r = lanes.getexp(t)
    assert r.is_cuda and r.tolist() == [2.0, -1074.0]
    mag, c, s = lanes.polar(3.0, 4.0)
    assert float(mag) == 5.0 and float(c) == 0.6 and float(s) == 0.8
    lanes.assert_fp_env(0)


def test_empty_inputs():
    from paper_2005_07403_b200 import svd2
    assert lanes.fma(np.zeros(0), np.zeros(0), np.zeros(0)).shape == (0,)
    tri = svd2.triangular_svd(np.zeros(0), np.zeros(0), np.zeros(0))
    assert tri.smax_scaled.shape == (0,)
