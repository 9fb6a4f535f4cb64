"""Lane primitives on the GPU (drop-in for lanesvd.lanes).

The reference builds its pipeline from elementwise NumPy/numba helpers
(lanes.py:69-259).  Here the same primitives are the device functions of
``csrc/b2s_lane.cuh`` that every kernel is built from; this module exposes
them with the reference's names and semantics through one elementwise
kernel (C-ABI ``b2s_lane_op``), so results are bit-identical to lanesvd's
for every input (NaN payload bits aside).  Arguments broadcast like NumPy
operands; host inputs give host (NumPy) results, CUDA tensors stay on their
device.  There is no CPU path: a call without the library raises.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .layout import LANE_WIDTH, is_device_array

__all__ = [
    "LANE_WIDTH", "DBL_MAX", "DBL_MIN_NORMAL", "DBL_TRUE_MIN", "EPS",
    "fma", "fnma", "relaxed_min", "relaxed_max", "select",
    "getexp", "scalef", "hypot_lane", "invsqrt_lane",
    "bit_and", "bit_or", "bit_xor", "bit_andnot",
    "fabs", "negate", "sign_mask",
    "complex_mul", "phase_from_parts", "polar",
    "assert_fp_env",
]

DBL_MAX = 1.7976931348623157e+308
DBL_MIN_NORMAL = 2.2250738585072014e-308
DBL_TRUE_MIN = 5e-324
EPS = 2.0 ** -53

_OPS = {"fma": 0, "fnma": 1, "relaxed_min": 2, "relaxed_max": 3, "select": 4, "getexp": 5,
        "scalef": 6, "hypot_lane": 7, "invsqrt_lane": 8, "bit_and": 9, "bit_or": 10,
        "bit_xor": 11, "bit_andnot": 12, "fabs": 13, "negate": 14, "sign_mask": 15,
        "complex_mul": 16, "phase_from_parts": 17, "polar": 18}


def _run(name, args, n_out):
    import torch
    dev = next((a.device for a in args if is_device_array(a)), None)
    host = dev is None
    if host:
        dev = torch.device("cuda", torch.cuda.current_device())
        arrs = np.broadcast_arrays(*[np.asarray(a, dtype=np.float64) for a in args])
        shape = arrs[0].shape
        ts = [torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(dev) for a in arrs]
    else:
        ts = [a if is_device_array(a) else torch.as_tensor(np.asarray(a, dtype=np.float64))
              for a in args]
        ts = [t.to(device=dev, dtype=torch.float64) for t in ts]
        ts = torch.broadcast_tensors(*ts)
        shape = tuple(ts[0].shape)
        ts = [t.reshape(-1).contiguous() for t in ts]
    n = int(ts[0].numel())
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(n_out)]
    if n == 0:                                   # nothing to launch (empty tensors have no storage)
        res = [o.cpu().numpy().reshape(shape) if host else o.reshape(shape) for o in outs]
        return res[0] if n_out == 1 else tuple(res)
    pi, _k1 = _lib.ptr_array([t.data_ptr() for t in ts])
    po, _k2 = _lib.ptr_array([t.data_ptr() for t in outs])
    with torch.cuda.device(dev):
        rc = _lib.lib.b2s_lane_op(_OPS[name], n, len(ts), pi, n_out, po,
                                  torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(rc, "b2s_lane_op(%s)" % name)
    if host:
        res = [o.cpu().numpy().reshape(shape) for o in outs]
    else:
        res = [o.reshape(shape) for o in outs]
    return res[0] if n_out == 1 else tuple(res)


def fma(a, b, c):
    """``a*b + c`` with a single rounding (lanes.py:69-83)."""
    return _run("fma", (a, b, c), 1)


def fnma(a, b, c):
    """``c - a*b`` with a single rounding (lanes.py:86-95)."""
    return _run("fnma", (a, b, c), 1)


def relaxed_min(a, b):
    """``a`` where ``a < b``, else ``b`` (lanes.py:102-110)."""
    return _run("relaxed_min", (a, b), 1)


def relaxed_max(a, b):
    """``a`` where ``a > b``, else ``b`` (lanes.py:113-115)."""
    return _run("relaxed_max", (a, b), 1)


def select(mask, a, b):
    """``b`` where ``mask`` is set, ``a`` elsewhere (lanes.py:117-119)."""
    m = mask if is_device_array(mask) else np.asarray(mask, dtype=bool)
    m = m.double() if is_device_array(m) else m.astype(np.float64)
    return _run("select", (m, a, b), 1)


def getexp(a):
    """floor(log2|a|) as float64, exact for subnormals; 0 -> -inf,
    +-inf -> +inf, NaN propagates (lanes.py:126-140)."""
    return _run("getexp", (a,), 1)


def scalef(a, e):
    """``a * 2**floor(e)`` with a single rounding (lanes.py:143-159)."""
    return _run("scalef", (a, e), 1)


def hypot_lane(a, b):
    """sqrt(a*a + b*b) without undue overflow (lanes.py:213-227)."""
    return _run("hypot_lane", (a, b), 1)


def invsqrt_lane(a):
    """``1 / sqrt(a)``, two correctly rounded operations (lanes.py:230-232)."""
    return _run("invsqrt_lane", (a,), 1)


def bit_and(a, b):
    return _run("bit_and", (a, b), 1)


def bit_or(a, b):
    return _run("bit_or", (a, b), 1)


def bit_xor(a, b):
    return _run("bit_xor", (a, b), 1)


def bit_andnot(a, b):
    """``~a & b`` on the raw lane patterns."""
    return _run("bit_andnot", (a, b), 1)


def fabs(x):
    """Clear the sign bit (lanes.py:169-206 sign algebra)."""
    return _run("fabs", (x,), 1)


def negate(x):
    return _run("negate", (x,), 1)


def sign_mask(x):
    """The sign bit as a +-0.0 pattern."""
    return _run("sign_mask", (x,), 1)


def complex_mul(ar, ai, br, bi):
    """(fma(ar, br, -(ai*bi)), fma(ar, bi, ai*br)) (lanes.py:235-245)."""
    return _run("complex_mul", (ar, ai, br, bi), 2)


def phase_from_parts(re, im, mag):
    """Unit phase (cos, sin) of re + i*im given its magnitude
    (lanes.py:248-259)."""
    return _run("phase_from_parts", (re, im, mag), 2)


def polar(zr, zi):
    """Magnitude and unit phase (cos, sin) of zr + i*zi."""
    return _run("polar", (zr, zi), 3)


def assert_fp_env(device=0):
    """The reference's floating-point environment canary (lanes.py:274-302),
    evaluated by the GPU's own FP64 units: round-to-nearest-even, gradual
    underflow, fused fma.  Raises if the environment is wrong."""
    _lib.assert_device_fp_env(int(device))
