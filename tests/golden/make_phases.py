"""Golden inputs and outputs of the REFERENCE's per-phase svd2 functions
(svd2.py:134-474), for the device phase entry points (b2s_svd2_phase,
tests/test_gpu_phases.py).  Build container only.

Two kinds of calls per field:
* "chain": the reference's own pipeline run phase by phase on every lane set
  of lanes.npz (patterned extremes, full-range bit-pattern fuzz, zeros and
  the first lanes of configs 2 and 4; up to 512 lanes each), each phase's
  actual inputs and outputs;
* "free": each phase on independent random finite inputs (wide exponents,
  signed zeros, equal values) that no pipeline would produce -- the phase
  functions are defined for any finite input.

Run:  python tests/golden/make_phases.py
"""

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from lanesvd import svd2  # noqa: E402


def flat(vals):
    """Values (arrays, (re, im|None) pairs, bool masks, tuples of those) ->
    one (k, n) float64 stack in order."""
    out = []

    def add(v):
        if isinstance(v, tuple):
            for x in v:
                if x is not None:
                    add(x)
        elif hasattr(v, "__dataclass_fields__"):
            for f in v.__dataclass_fields__:
                add(getattr(v, f))
        else:
            out.append(np.asarray(v, dtype=np.float64))
    for v in vals:
        add(v)
    return np.stack(out)


def chain(parts, rec, key):
    scale = svd2.compute_scale(parts)
    rec[key + "/compute_scale/in"] = flat([tuple(parts)])
    rec[key + "/compute_scale/out"] = flat([scale.shift, scale.parts])
    k = len(parts) // 4
    ent = [(scale.parts[i], None) for i in range(4)] if k == 1 else \
        [(scale.parts[2 * i], scale.parts[2 * i + 1]) for i in range(4)]
    norms = svd2.column_norms(*ent)
    rec[key + "/column_norms/in"] = flat([tuple(ent)])
    rec[key + "/column_norms/out"] = flat([norms])
    mags, n1, n2 = norms[:4], norms[4], norms[5]
    piv = svd2.column_pivot(tuple(ent), mags, n1, n2)
    rec[key + "/column_pivot/in"] = flat([tuple(ent), mags, n1, n2])
    rec[key + "/column_pivot/out"] = flat([piv])
    ent_p, mags_p, n1, n2, swap_c = piv
    rs = svd2.row_sort(ent_p, mags_p)
    rec[key + "/row_sort/in"] = flat([ent_p, mags_p])
    rec[key + "/row_sort/out"] = flat([rs])
    ent_s, mags_s, swap_r = rs
    lp = svd2.left_phase_reduce(*ent_s, mags_s[0], mags_s[1])
    rec[key + "/left_phase_reduce/in"] = flat([ent_s, mags_s[0], mags_s[1]])
    rec[key + "/left_phase_reduce/out"] = flat([lp])
    b11, b21, f12, f22, ph1, ph2 = lp
    gq = svd2.givens_qr(b11, b21, f12, f22, n1)
    rec[key + "/givens_qr/in"] = flat([b11, b21, f12, f22, n1])
    rec[key + "/givens_qr/out"] = flat([gq])
    g_tan, g_cos, r11, g12, g22 = gq
    pf = svd2.phase_fix_r(g12, g22)
    rec[key + "/phase_fix_r/in"] = flat([g12, g22])
    rec[key + "/phase_fix_r/out"] = flat([pf])
    r12, r22, dt, dh = pf
    tri = svd2.triangular_svd(r11, r12, r22)
    rec[key + "/triangular_svd/in"] = flat([r11, r12, r22])
    rec[key + "/triangular_svd/out"] = flat([tri])
    urv = svd2.UrvState(swap_cols=swap_c, swap_rows=swap_r, row_phase1=ph1, row_phase2=ph2,
                        givens_tan=g_tan, givens_cos=g_cos, r12_phase=dt, r22_phase=dh,
                        r11=r11, r12=r12, r22=r22)
    for name, fn in (("assemble_uv", svd2.assemble_uv), ("assemble_uv_sine", svd2.assemble_uv_sine)):
        out = fn(urv, tri, scale.shift)
        rec[key + "/%s/in" % name] = flat([urv, tri, scale.shift])
        rec[key + "/%s/out" % name] = flat([out])


def rnd(rng, n, lo=-1000, hi=1000, zeros=0.1):
    x = np.ldexp(rng.uniform(1, 2, n) * np.where(rng.random(n) < 0.5, -1.0, 1.0),
                 rng.integers(lo, hi, n))
    x[rng.random(n) < zeros] = 0.0
    x[rng.random(n) < zeros / 2] = -0.0
    return x


def free(rng, cplx, rec, key, n=512):
    pos = lambda: np.abs(rnd(rng, n, -1000, 1021))
    val = lambda: (rnd(rng, n, -1000, 1021), rnd(rng, n, -1000, 1021) if cplx else None)
    ent = tuple(val() for _ in range(4))
    mags = tuple(pos() for _ in range(4))
    n1, n2 = pos(), pos()
    n2[::7] = n1[::7]                                 # ties keep the order
    calls = {
        "column_norms": (svd2.column_norms, ent),
        "column_pivot": (svd2.column_pivot, (ent, mags, n1, n2)),
        "row_sort": (svd2.row_sort, (ent, mags)),
        "left_phase_reduce": (svd2.left_phase_reduce, ent + (mags[0], mags[1])),
        "givens_qr": (svd2.givens_qr, (mags[0], mags[1], ent[2], ent[3], n1)),
        "phase_fix_r": (svd2.phase_fix_r, (ent[0], ent[1])),
    }
    if not cplx:
        calls["triangular_svd"] = (svd2.triangular_svd, (n1, mags[2], mags[3]))
    with np.errstate(all="ignore"):
        for name, (fn, args) in calls.items():
            rec[key + "/%s/in" % name] = flat(list(args))
            rec[key + "/%s/out" % name] = flat([fn(*args)])


def main():
    lanes = np.load(os.path.join(HERE, "lanes.npz"))
    rec = {}
    sets = {"patterned_real": 8, "patterned_complex": 8, "fuzz_real": 512, "fuzz_complex": 512,
            "zeros_real": 256, "zeros_complex": 256, "config2": 256, "config4": 256}
    for name, m in sets.items():
        re = lanes[name + "/in_re"][:, :m]
        im = lanes[name + "/in_im"][:, :m] if name + "/in_im" in lanes.files else None
        parts = tuple(re[t] for t in range(4)) if im is None else \
            tuple(x for t in range(4) for x in (re[t], im[t]))
        with np.errstate(all="ignore"):
            chain(parts, rec, "chain_" + name)
    free(np.random.default_rng(61), False, rec, "free_real")
    free(np.random.default_rng(62), True, rec, "free_complex")
    np.savez_compressed(os.path.join(HERE, "phases.npz"), **rec)
    print(len(rec), "arrays")


if __name__ == "__main__":
    main()
