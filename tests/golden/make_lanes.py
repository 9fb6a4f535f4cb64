"""Golden inputs and outputs of the REFERENCE's lane primitives
(lanesvd.lanes, lanes.py:69-259) for the device ops (b2s_lane_op,
tests/test_gpu_lanes.py).  Build container only.

Inputs mix full-range random bit patterns (normal, subnormal, zero,
infinite, NaN), wide-exponent finite values and the special values that
the reference's docstrings single out.

Run:  python tests/golden/make_lanes.py
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from lanesvd import lanes  # noqa: E402

SPECIAL = np.array([0.0, -0.0, 1.0, -1.0, 5e-324, -5e-324, 2.2250738585072014e-308,
                    1.7976931348623157e308, -1.7976931348623157e308, np.inf, -np.inf, np.nan,
                    0.5, 2.0 ** 1022, 2.0 ** -1022, 3.0, 1e-300, 1e300])


def sample(rng, n):
    bits = rng.integers(0, 2 ** 63, n, dtype=np.uint64) | (
        rng.integers(0, 2, n, dtype=np.uint64) << np.uint64(63))
    a = bits.view(np.float64).copy()
    w = np.ldexp(rng.uniform(1, 2, n) * np.where(rng.random(n) < 0.5, -1.0, 1.0),
                 rng.integers(-1074, 1024, n))
    pick = rng.random(n)
    a = np.where(pick < 0.4, w, a)
    s = rng.integers(0, len(SPECIAL), n)
    a = np.where(pick > 0.9, SPECIAL[s], a)
    return a


def main():
    rng = np.random.default_rng(71)
    n = 4096
    X = [sample(rng, n) for _ in range(4)]
    mask = rng.random(n) < 0.5
    e = np.where(rng.random(n) < 0.8, rng.uniform(-3000, 3000, n), sample(rng, n))
    calls = {
        "fma": (X[0], X[1], X[2]), "fnma": (X[0], X[1], X[2]),
        "relaxed_min": (X[0], X[1]), "relaxed_max": (X[0], X[1]),
        "select": (mask, X[0], X[1]), "getexp": (X[0],), "scalef": (X[0], e),
        "hypot_lane": (X[0], X[1]), "invsqrt_lane": (np.abs(X[2]),),
        "bit_and": (X[0], X[1]), "bit_or": (X[0], X[1]), "bit_xor": (X[0], X[1]),
        "bit_andnot": (X[0], X[1]), "fabs": (X[0],), "negate": (X[0],), "sign_mask": (X[0],),
        "complex_mul": tuple(X), "phase_from_parts": (X[0], X[1], np.abs(X[2])),
        "polar": (X[0], X[1]),
    }
    out = {}
    with np.errstate(all="ignore"):
        for name, args in calls.items():
            r = getattr(lanes, name)(*args)
            r = r if isinstance(r, tuple) else (r,)
            out[name + "/in"] = np.stack([np.asarray(a, dtype=np.float64) for a in args])
            out[name + "/out"] = np.stack([np.asarray(x, dtype=np.float64) for x in r])
    np.savez_compressed(os.path.join(HERE, "lanes_ops.npz"), **out)
    print(sorted({k.split("/")[0] for k in out}))


if __name__ == "__main__":
    main()
