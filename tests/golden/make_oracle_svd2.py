"""Golden outputs of the REFERENCE's independent double-double SVD,
lanesvd.verify.oracle_svd2 (verify.py:259-352), for the GPU port
(b2s_oracle_svd2, tests/test_gpu_verify.py).  Build container only.

Inputs: the reference's own test matrices (test_verify.py:98-186: the worked
example, a diagonal, rank one, zero, 2^+-200-scaled real and complex normal
matrices) plus seeded wide-range real and complex matrices with exact zeros.

Run:  python tests/golden/make_oracle_svd2.py
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from lanesvd import verify  # noqa: E402


def words(res):
    dd = lambda d: [d.hi, d.lo]
    out = dd(res.smax) + dd(res.smin)
    for e in (res.u11, res.u21, res.u12, res.u22, res.v11, res.v21, res.v12, res.v22):
        out += dd(e[0]) + dd(e[1])
    return np.stack(out)


def wide(rng, n, cplx):
    e = rng.integers(-1000, 1000, size=(n, 2, 2))
    m = rng.uniform(1, 2, size=(n, 2, 2)) * np.where(rng.random((n, 2, 2)) < 0.5, -1.0, 1.0)
    x = np.ldexp(m, e)
    x[rng.random((n, 2, 2)) < 0.1] = 0.0
    if cplx:
        y = np.ldexp(rng.uniform(1, 2, size=(n, 2, 2)), rng.integers(-1000, 1000, size=(n, 2, 2)))
        y[rng.random((n, 2, 2)) < 0.1] = 0.0
        x = x + 1j * y
    return x


def main():
    rng = np.random.default_rng(54)
    sets = {
        "worked": np.array([[[4.0, 2.0], [3.0, -1.0]]]),
        "diagonal": np.array([[[3.0, 0.0], [0.0, -2.0]]]),
        "rank_one": np.array([[[1.0, 1.0], [0.0, 0.0]]]),
        "zero": np.zeros((1, 2, 2)),
        "real_scaled": rng.standard_normal((64, 2, 2)) * np.exp2(rng.integers(-200, 200, (64, 1, 1))),
        "complex_normal": (np.random.default_rng(55).standard_normal((32, 2, 2))
                           + 1j * np.random.default_rng(56).standard_normal((32, 2, 2))),
        "real_wide": wide(np.random.default_rng(57), 4096, False),
        "complex_wide": wide(np.random.default_rng(58), 4096, True),
    }
    out = {}
    for name, mats in sets.items():
        out[name + "/in"] = mats
        out[name + "/out"] = words(verify.oracle_svd2(mats))
    np.savez_compressed(os.path.join(HERE, "oracle_svd2.npz"), **out)
    print(sorted(out))


if __name__ == "__main__":
    main()
