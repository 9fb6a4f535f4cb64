"""The rest of svd2_lanes' with_states tuple from the REFERENCE ITSELF
(build container only): for every lane set of lanes.npz that carries a
state dump, lanesvd.svd2.svd2_lanes(parts, with_states=True)
(svd2.py:521-570) is run on the same inputs and the trains the dump does not
hold -- TriangleSvd left/right sec2 and cos (svd2.py:90-105) and
ScaleResult.parts (svd2.py:61-65) -- are stored in states_full.npz.

Run:  python tests/golden/make_states_full.py
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from lanesvd import svd2  # noqa: E402


def main():
    lanes = np.load(os.path.join(HERE, "lanes.npz"))
    out = {}
    for key in lanes.files:
        rec, name = key.split("/", 1)
        if name != "states":
            continue
        re = lanes[rec + "/in_re"]
        im = lanes[rec + "/in_im"] if rec + "/in_im" in lanes.files else None
        parts = tuple(re[t] for t in range(4)) if im is None else \
            tuple(x for t in range(4) for x in (re[t], im[t]))
        _, scale, _, tri = svd2.svd2_lanes(parts, with_states=True)
        out[rec + "/tri"] = np.stack([tri.left_sec2, tri.left_cos, tri.right_sec2, tri.right_cos])
        out[rec + "/scaled_parts"] = np.stack(scale.parts)
    np.savez_compressed(os.path.join(HERE, "states_full.npz"), **out)
    print(sorted(out))


if __name__ == "__main__":
    main()
