"""Per-lane 8-eps gate counts from the REFERENCE's own verifier (build
container only; the reference cannot travel).

lanesvd.verify.metrics (verify.py:395-477) computes per-lane double-double
rho, delta, eta and returns only their maxima; this script wraps its
``_dd_max`` to see the per-lane values it reduces, and counts the lanes
whose rho, delta or eta exceeds 8 eps (eps = 2^-52, the north_star gate) --
on the reference's own outputs for config 1 (all 2^20 lanes) and the
config-3 / config-4 parity windows of digests.json.  The engine's outputs
are bit-identical, so its count (the GPU verifier's over_8eps_frobenius,
tests/test_gpu_verify.py) must equal these.

Run:  python tests/golden/make_quality_counts.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from lanesvd import driver, layout, verify  # noqa: E402

from paper_2005_07403_b200 import synth  # noqa: E402

TOL = 2.0 ** -49


def over(dd):
    return (dd.hi > TOL) | ((dd.hi == TOL) & (dd.lo > 0))


def counts(config, seed, lo, n):
    re, im = synth.generate(config, seed, lo, n)
    b = layout.from_trains(re, im)
    out, _ = driver.run_batch(b, driver.RunConfig(field=b.field))
    seen = []
    orig = verify._dd_max
    verify._dd_max = lambda a: (seen.append(a), orig(a))[1]
    try:
        verify.metrics(b, out)
    finally:
        verify._dd_max = orig
    rho, delta, eta = seen          # metrics reduces rho, delta, eta in this order
    bad = over(rho) | over(delta) | over(eta)
    return int(np.count_nonzero(bad[:n]))


def main():
    with open(os.path.join(HERE, "digests.json")) as fh:
        dg = json.load(fh)
    seed, W = dg["seed"], dg["window"]
    res = {"seed": seed, "tolerance": "8 * 2^-52 on rho, delta, eta (Frobenius), double-double",
           "how": "lanesvd.verify.metrics per-lane values (via its _dd_max)", "sets": {}}
    res["sets"]["config1_full"] = {"config": 1, "windows": [[0, 1 << 20]],
                                   "over_8eps_frobenius": counts(1, seed, 0, 1 << 20)}
    for config in (3, 4):
        wins = [w["lo"] for w in dg["configs"][str(config)]["windows"]]
        total = sum(counts(config, seed, lo, W) for lo in wins)
        res["sets"]["config%d_windows" % config] = {
            "config": config, "windows": [[lo, W] for lo in wins], "over_8eps_frobenius": total}
        print(config, total, flush=True)
    with open(os.path.join(HERE, "quality_counts.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res["sets"]["config1_full"]))


if __name__ == "__main__":
    main()
