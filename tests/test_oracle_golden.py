"""Pin the CPU oracle (oracle/svd2_oracle.c) to the reference's own outputs.

tests/golden/ was produced by running the reference lanesvd itself
(tests/golden/make_golden.py); every comparison here is bit-for-bit.  The
known-answer tests restate the reference's own unit-test vectors
(pkg/tests/test_svd2.py, test_driver.py) against the oracle.
"""

import numpy as np
import pytest

import oracle
from helpers import assert_bits_equal, bits, digest
from paper_2005_07403_b200 import synth

DBL_MAX = 1.7976931348623157e308
TRUE_MIN = 5e-324
EPS = 2.0 ** -53

RECORD_MODES = {"patterned_real_safe": ("safe", False),
                "fuzz_real_safe": ("safe", False),
                "fuzz_real_unc": ("unconditional", False),
                "fuzz_real_sine": ("none", True),
                "fuzz_complex_sine": ("none", True)}


def _run_record(rec, name):
    mode, sine = RECORD_MODES.get(name, ("none", False))
    return oracle.svd2(rec["in_re"], rec.get("in_im"), backscale_mode=mode,
                       sine_form=sine, with_states="states" in rec)


def test_oracle_matches_reference_lane_records(lanes):
    assert len(lanes) >= 15
    for name, rec in lanes.items():
        out = _run_record(rec, name)
        for k, arr in out.trains().items():
            assert_bits_equal(arr, rec[k], "%s/%s" % (name, k))
        if "states" in rec:
            assert_bits_equal(out.states, rec["states"], name + "/states")


@pytest.mark.parametrize("config", [0, 1, 2])
def test_oracle_matches_reference_full_configs(digests, config):
    entry = digests["configs"][str(config)]
    re, im = synth.generate(config, digests["seed"], 0, entry["n"])
    assert digest(re) == entry["input"]["re"]
    if im is not None:
        assert digest(im) == entry["input"]["im"]
    for key in ("none", "safe", "unconditional", "sine"):
        if key not in entry:
            continue
        mode = key if key in ("safe", "unconditional") else "none"
        out = oracle.svd2(re, im, backscale_mode=mode, sine_form=key == "sine")
        got = {k: digest(v) for k, v in out.trains().items()}
        assert got == entry[key], (config, key)


@pytest.mark.parametrize("config", [3, 4])
def test_oracle_matches_reference_windows(digests, config):
    entry = digests["configs"][str(config)]
    W = digests["window"]
    for w in entry["windows"][:6]:
        re, im = synth.generate(config, digests["seed"], w["lo"], W)
        assert digest(re) == w["input"]["re"]
        out = oracle.svd2(re, im)
        got = {k: digest(v) for k, v in out.trains().items()}
        assert got == w["none"], (config, w["lo"])


# ---------------------------------------------------------------------------
# known answers from the reference's unit tests
# ---------------------------------------------------------------------------

def _real(mats, **kw):
    a = np.asarray(mats, dtype=np.float64).reshape(-1, 2, 2)
    re = np.stack([a[:, 0, 0], a[:, 1, 0], a[:, 0, 1], a[:, 1, 1]])
    return oracle.svd2(re, **kw)


def _u(out, k):
    u = out.u_re
    return np.array([[u[0, k], u[2, k]], [u[1, k], u[3, k]]])


def _v(out, k):
    v = out.v_re
    return np.array([[v[0, k], v[2, k]], [v[1, k], v[3, k]]])


def test_kat_scaling_shifts():
    # test_svd2.py:64-116
    out = _real([[[1, 0], [0, 1]], [[DBL_MAX, DBL_MAX], [DBL_MAX, -DBL_MAX]],
                 [[0, 0], [0, 0]], [[TRUE_MIN, 0.0], [0.0, DBL_MAX]]])
    assert out.shift.tolist() == [1021.0, -2.0, DBL_MAX, -2.0]
    assert out.smax[0] == 2.0 ** 1021
    c = oracle.svd2(np.array([[3.0], [0], [0], [0]]), np.array([[4.0], [0], [0], [0]]))
    assert c.shift[0] == 1019.0


def test_kat_worked_example():
    # test_svd2.py:363-383: A = [[4,2],[3,-1]]
    out = _real([[4, 2], [3, -1]])
    assert out.shift[0] == 1019.0
    smax, smin, sh = oracle.backscale(out.smax, out.smin, out.shift, "safe")
    assert abs(smax[0] - 5.116672736016927) <= 1e-6 * 5.116672736016927
    assert abs(smin[0] - 1.954395075848548) <= 1e-6 * 1.954395075848548
    assert np.signbit(sh[0]) and sh[0] == 0.0
    u, v = _u(out, 0), _v(out, 0)
    assert abs(u[0, 0] - 0.8506508083520399) <= 1e-6
    assert abs(u[1, 0] - 0.5257311121191336) <= 1e-6
    assert abs(v[0, 0] - 0.9732489894677302) <= 1e-6
    assert abs(v[1, 0] - 0.22975292054736118) <= 1e-6
    rec = u @ np.diag([smax[0], smin[0]]) @ v.T
    assert np.abs(rec - [[4, 2], [3, -1]]).max() <= 1e-13


def test_kat_identity_and_zero_lanes():
    out = _real([[[1, 0], [0, 1]], [[0, 0], [0, 0]]])
    assert _u(out, 0).tolist() == [[1, 0], [0, 1]]
    assert _v(out, 0).tolist() == [[1, 0], [0, 1]]
    assert out.smax[1] == 0.0 and out.shift[1] == DBL_MAX
    # SURVEY Appendix A special-lane table: U = [[1,-0],[0,1]] pattern
    assert bits(out.u_re[:, 1]).tolist() == bits([1.0, 0.0, -0.0, 1.0]).tolist()


def test_kat_row_and_column_swap_symmetries():
    base = _real([[4, 2], [3, -1]])
    rows = _real([[3, -1], [4, 2]])
    cols = _real([[2, 4], [-1, 3]])
    assert_bits_equal(rows.u_re[[1, 0, 3, 2]], base.u_re)
    assert_bits_equal(rows.v_re, base.v_re)
    assert_bits_equal(cols.v_re[[1, 0, 3, 2]], base.v_re)
    assert_bits_equal(cols.u_re, base.u_re)


def test_kat_triangle_rank_one():
    # test_svd2.py:298-306 / test_acceptance patterned rank-1 lane
    out = _real([[1, 1], [0, 0]])
    assert out.smin[0] == 0.0
    assert out.smax[0] == 1.4142135623730949 * 2.0 ** 1021


def test_kat_backscale_boundaries():
    # test_svd2.py:478-536
    bs = oracle.backscale
    m, n_, s = bs([2.0 ** 1020], [2.0 ** 1000], [-10.0], "unconditional")
    assert np.isinf(m[0]) and n_[0] == 2.0 ** 1010 and np.signbit(s[0])
    m, n_, s = bs([2.0 ** 1022], [1.0], [-1.0], "safe")
    assert m[0] == 2.0 ** 1023 and np.signbit(s[0])
    m, n_, s = bs([2.0 ** 1022], [1.0], [-2.0], "safe")
    assert m[0] == 2.0 ** 1022 and s[0] == -2.0
    m, n_, s = bs([1.0], [1.0], [1022.0], "safe")
    assert n_[0] == 2.0 ** -1022 and np.signbit(s[0])
    m, n_, s = bs([1.0], [1.0], [1023.0], "safe")
    assert n_[0] == 1.0 and s[0] == 1023.0
    m, n_, s = bs([1.0], [0.0], [1023.0], "safe")
    assert m[0] == 2.0 ** -1023 and n_[0] == 0.0 and np.signbit(s[0])
    m, n_, s = bs([0.0], [0.0], [DBL_MAX], "safe")
    assert m[0] == 0.0 and np.signbit(s[0])


def test_kat_backscale_modes_on_diag():
    # test_driver.py:190-213
    mats = np.stack([np.diag([1e300, 1e-310]), np.diag([3.0, 1.0])])
    none = _real(mats)
    safe = _real(mats, backscale_mode="safe")
    unc = _real(mats, backscale_mode="unconditional")
    assert safe.smax[1] == 3.0 and safe.smin[1] == 1.0
    assert safe.shift[0] == none.shift[0] != 0.0
    assert unc.smax[0] == 1e300 and unc.smin[0] == 1e-310


def test_kat_primitives():
    # test_lanes.py: getexp, scalef, hypot, invsqrt exact cases
    assert oracle.getexp(2.0 ** -1074) == -1074
    assert oracle.getexp(0.0) == -np.inf
    assert oracle.getexp(3.0) == 1.0
    assert oracle.scalef(1.0, 2.7) == 4.0
    assert oracle.scalef(3.0, -1076) == TRUE_MIN
    assert oracle.scalef(1.0, -1076) == 0.0
    assert oracle.scalef(2.0, -1075) == TRUE_MIN
    assert oracle.hypot(3.0, 4.0) == 5.0
    assert oracle.hypot(2.0 ** 1022, 2.0 ** 1022) == np.sqrt(2.0) * 2.0 ** 1022
    assert oracle.invsqrt(4.0) == 0.5


def test_oracle_thread_count_invariance():
    re, _ = synth.generate(0, 5, 0, 4096)
    a = oracle.svd2(re, threads=1)
    b = oracle.svd2(re, threads=7)
    for k in a.trains():
        assert_bits_equal(a.trains()[k], b.trains()[k], k)


def test_oracle_states_invariants():
    # test_acceptance.py:115-140 Theorem-1 invariants on the state dump
    rng = np.random.default_rng(3)
    re = rng.standard_normal((4, 8192)) * np.exp2(rng.integers(-300, 300, (4, 8192)))
    out = oracle.svd2(re, with_states=True)
    st = out.states
    lt, rt, rc = st[12], st[13], 1.0 / np.sqrt(1.0 + st[13] ** 2)
    assert (np.abs(lt) <= 1.0).all()
    assert (np.abs(rt) <= np.sqrt(2.0) * (1 + 2 * EPS)).all()
    assert (np.abs(rt) >= np.abs(lt)).all()
    assert (out.smax >= out.smin).all() and (out.smin >= 0).all()
    assert np.isfinite(st).all()


def test_train_checksum_numpy_and_torch_agree():
    """The position-keyed checksums of the full-size golden file: the NumPy
    form (reference side) and the torch form (device side) are one function."""
    import torch
    from helpers import train_checksum_np, train_checksum_torch
    rng = np.random.default_rng(5)
    x = rng.standard_normal(10_000) * 1e300
    x[::7] = -0.0
    for lane0 in (0, 12345, (1 << 30) - 10_000):
        assert train_checksum_np(x, lane0) == train_checksum_torch(torch.from_numpy(x), lane0)
    y = x.copy()
    y[5000] = np.nextafter(y[5000], np.inf)
    assert train_checksum_np(y, 0) != train_checksum_np(x, 0)
