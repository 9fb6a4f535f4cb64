"""Generate the golden fixtures from the REFERENCE ITSELF (build container only).

Imports the reference package ``lanesvd`` read-only from
/root/reference/pkg/src (it cannot travel to the GPU box), runs its own
``driver.run_batch`` on seeded inputs, and commits:

* ``digests.json`` -- SHA-256 of every output train of the reference for the
  full BASELINE configs 0 (n=65536), 1 (n=2^20) and 2 (n=2^24), for the three
  backscale modes and the sine form on config 0, and for seeded parity
  windows of the large configs 3 (n=2^30) and 4 (n=2^28); inputs regenerate
  bit-identically from ``paper_2005_07403_b200.synth`` (host or device).
* ``lanes.npz`` -- full input/output bit patterns for small lane sets: the
  acceptance suite's patterned extreme lanes, full-range random bit-pattern
  fuzz lanes (real and complex, via lanesvd.cli.random_finite), the first
  lanes of each config, and state dumps (driver._dump_states order).

Run:  python tests/golden/make_golden.py   (takes a few minutes on 8 cores)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import lanesvd  # noqa: E402
from lanesvd import cli, driver, layout  # noqa: E402

from paper_2005_07403_b200 import synth  # noqa: E402

SEED = 20250705
DBL_MAX = 1.7976931348623157e308
TRUE_MIN = 5e-324
WINDOW = 1 << 15


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64)
                          .view(np.uint64).tobytes()).hexdigest()


def out_digests(out):
    d = {"u_re": digest(out.u_re), "v_re": digest(out.v_re),
         "smax": digest(out.smax), "smin": digest(out.smin),
         "shift": digest(out.shift)}
    if out.u_im is not None:
        d["u_im"] = digest(out.u_im)
        d["v_im"] = digest(out.v_im)
    return d


class _Cat:
    pass


def ref_run(re, im, mode="none", sine=False, threads=0, piece=1 << 21):
    """Reference run_batch, in contiguous 2^21-lane sub-batches for large n
    (outputs are partition-invariant, test_driver.py:165-177)."""
    n = re.shape[1]
    outs = []
    for lo in range(0, max(n, 1), piece):
        hi = min(n, lo + piece)
        b = layout.from_trains(re[:, lo:hi], None if im is None else im[:, lo:hi])
        cfg = driver.RunConfig(field=b.field, backscale_mode=mode,
                               threads=threads)
        out, _ = driver.run_batch(b, cfg, sine_form=sine)
        outs.append(out)
    if len(outs) == 1:
        return outs[0]
    cat = _Cat()
    for k in ("u_re", "u_im", "v_re", "v_im"):
        parts = [getattr(o, k) for o in outs]
        setattr(cat, k, None if parts[0] is None else np.concatenate(parts, axis=1))
    for k in ("smax", "smin", "shift"):
        setattr(cat, k, np.concatenate([getattr(o, k) for o in outs]))
    return cat


def windows(config, n, count, seed):
    """Seeded window starts (multiples of 256) plus the first and last."""
    rng = np.random.default_rng(seed + config)
    starts = sorted(set([0, n - WINDOW] + [int(x) * 256 for x in rng.integers(
        0, (n - WINDOW) // 256, count)]))
    return starts


def patterned():
    # test_acceptance.py:38-49 patterned extreme lanes
    return np.array([
        [[DBL_MAX, DBL_MAX], [DBL_MAX, -DBL_MAX]],
        [[1.0, 0.0], [0.0, 1.0]],
        [[0.0, 0.0], [0.0, 0.0]],
        [[TRUE_MIN, -TRUE_MIN], [TRUE_MIN, TRUE_MIN]],
        [[DBL_MAX, 0.0], [0.0, TRUE_MIN]],
        [[1.0, 1.0], [0.0, 0.0]],
        [[-DBL_MAX, TRUE_MIN], [0.0, 1.0]],
        [[2.0 ** -1022, 2.0 ** 1023], [-0.0, 2.0 ** -1074]],
    ])


def to_trains(mats):
    order = ((0, 0), (1, 0), (0, 1), (1, 1))
    return np.stack([mats[:, i, j] for (i, j) in order])


def lane_record(prefix, re, im, store, mode="none", sine=False, states=True):
    out = ref_run(re, im, mode=mode, sine=sine, threads=1)
    store[prefix + "/in_re"] = re
    if im is not None:
        store[prefix + "/in_im"] = im
    for k, v in out_digests(out).items():
        store[prefix + "/" + k] = np.asarray(getattr(out, k))
    if states:
        with tempfile.NamedTemporaryFile(suffix=".bin") as fh:
            b = layout.from_trains(re, im)
            driver.run_batch(b, driver.RunConfig(field=b.field, threads=1),
                             sine_form=sine, dump_states_to=fh.name)
            data = np.fromfile(fh.name, dtype="<f8")
        store[prefix + "/states"] = data.reshape(-1, b.n_hat)


def main():
    dig = {"seed": SEED, "window": WINDOW, "reference": "lanesvd " +
           lanesvd.__version__, "configs": {}}
    # full configs 0-2
    for config in (0, 1, 2):
        n = synth.CONFIGS[config]["n"]
        re, im = synth.generate(config, SEED, 0, n)
        entry = {"n": n, "input": {"re": digest(re)}}
        if im is not None:
            entry["input"]["im"] = digest(im)
        entry["none"] = out_digests(ref_run(re, im))
        if config == 0:
            entry["safe"] = out_digests(ref_run(re, im, mode="safe"))
            entry["unconditional"] = out_digests(
                ref_run(re, im, mode="unconditional"))
            entry["sine"] = out_digests(ref_run(re, im, sine=True))
        if config == 2:
            entry["safe"] = out_digests(ref_run(re, im, mode="safe"))
        dig["configs"][str(config)] = entry
        print("config", config, "done", flush=True)
    # windows of the large configs
    for config, count in ((3, 14), (4, 14)):
        n = synth.CONFIGS[config]["n"]
        ws = []
        for lo in windows(config, n, count, SEED):
            re, im = synth.generate(config, SEED, lo, WINDOW)
            d = {"lo": lo, "input": {"re": digest(re)}}
            if im is not None:
                d["input"]["im"] = digest(im)
            d["none"] = out_digests(ref_run(re, im))
            ws.append(d)
        dig["configs"][str(config)] = {"n": n, "windows": ws}
        print("config", config, "windows done", flush=True)
    with open(os.path.join(HERE, "digests.json"), "w") as fh:
        json.dump(dig, fh, indent=1, sort_keys=True)

    store = {}
    pat = to_trains(patterned())
    pat_pad = np.zeros((4, 8))
    pat_pad[:, :pat.shape[1]] = pat
    lane_record("patterned_real", pat_pad, None, store)
    lane_record("patterned_real_safe", pat_pad, None, store, mode="safe",
                states=False)
    lane_record("patterned_complex", pat_pad, np.zeros((4, 8)), store)
    rng = np.random.default_rng(SEED)
    fr = cli.random_finite(rng, 4 * 2048).reshape(4, 2048)
    lane_record("fuzz_real", fr, None, store)
    fc = cli.random_finite(rng, 8 * 2048).reshape(8, 2048)
    lane_record("fuzz_complex", fc[0::2], fc[1::2], store)
    # zero-heavy fuzz: random patterns with ~30% exact (+-)zeros
    zr = cli.random_finite(rng, 4 * 1024).reshape(4, 1024)
    zr[rng.random(zr.shape) < 0.3] = 0.0
    zr[rng.random(zr.shape) < 0.05] = -0.0
    lane_record("zeros_real", zr, None, store)
    zc = cli.random_finite(rng, 8 * 1024).reshape(8, 1024)
    zc[rng.random(zc.shape) < 0.3] = 0.0
    lane_record("zeros_complex", zc[0::2], zc[1::2], store)
    lane_record("fuzz_real_sine", fr[:, :512], None, store, sine=True,
                states=False)
    lane_record("fuzz_complex_sine", fc[0::2, :512], fc[1::2, :512], store,
                sine=True, states=False)
    lane_record("fuzz_real_safe", fr[:, :512], None, store, mode="safe",
                states=False)
    lane_record("fuzz_real_unc", fr[:, :512], None, store,
                mode="unconditional", states=False)
    for config, m in ((0, 256), (1, 256), (2, 1024), (4, 1024)):
        re, im = synth.generate(config, SEED, 0, m)
        lane_record("config%d" % config, re, im, store, states=False)
    np.savez_compressed(os.path.join(HERE, "lanes.npz"), **store)
    print("wrote", len(store), "arrays")
    write_metrics()


def _mstr(x):
    import mpmath
    with mpmath.workprec(240):
        return mpmath.nstr(x, 80)


def write_metrics():
    """Reference verify.metrics (double-double) for GPU-verifier parity."""
    from lanesvd import verify
    res = {}
    data = np.load(os.path.join(HERE, "lanes.npz"))
    recs = {}
    for key in data.files:
        rec, name = key.split("/", 1)
        recs.setdefault(rec, {})[name] = data[key]
    for name in ("fuzz_real", "fuzz_complex", "zeros_real", "zeros_complex",
                 "patterned_real", "patterned_real_safe", "fuzz_real_safe",
                 "fuzz_real_unc", "config2", "config4"):
        rec = recs[name]
        b = layout.from_trains(rec["in_re"], rec.get("in_im"))
        out = layout.SvdBatchOut(n=b.n, u_re=rec["u_re"], u_im=rec.get("u_im"),
                                 v_re=rec["v_re"], v_im=rec.get("v_im"),
                                 smax=rec["smax"], smin=rec["smin"], shift=rec["shift"])
        m = verify.metrics(b, out)
        res[name] = {"kappa": _mstr(m.kappa), "rho": _mstr(m.rho), "delta": _mstr(m.delta),
                     "eta": _mstr(m.eta), "excluded": m.rho_excluded_lanes}
    for config in (0, 1):
        n = synth.CONFIGS[config]["n"]
        re, im = synth.generate(config, SEED, 0, n)
        out = ref_run(re, im)
        b = layout.from_trains(re, im)
        o = layout.SvdBatchOut(n=n, u_re=out.u_re, u_im=out.u_im, v_re=out.v_re, v_im=out.v_im,
                               smax=out.smax, smin=out.smin, shift=out.shift)
        m = verify.metrics(b, o)
        res["config%d_full" % config] = {"kappa": _mstr(m.kappa), "rho": _mstr(m.rho),
                                         "delta": _mstr(m.delta), "eta": _mstr(m.eta),
                                         "excluded": m.rho_excluded_lanes}
        print("metrics config", config, res["config%d_full" % config], flush=True)
    with open(os.path.join(HERE, "metrics.json"), "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    if "--metrics-only" in sys.argv:
        write_metrics()
    else:
        main()
