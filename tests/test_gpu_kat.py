"""GPU: the reference's own unit-test assertions (lanesvd tests/test_svd2.py,
scaling through the full pipeline) run against this engine's svd2 module --
the per-phase device entry points and svd2_lanes -- with the reference's
known answers and tolerances."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2005_07403_b200 import lanes, svd2  # noqa: E402

DBL_MAX = 1.7976931348623157e308
TRUE_MIN = 5e-324
EPS = 2.0 ** -53


def a(x):
    return np.array([x], dtype=np.float64)


def bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def real(m):
    """Column-major component trains of one real 2x2 matrix (or a stack)."""
    m = np.asarray(m, dtype=np.float64).reshape(-1, 2, 2)
    return tuple(np.ascontiguousarray(m[:, i, j]) for i, j in ((0, 0), (1, 0), (0, 1), (1, 1)))


def cplx(m):
    m = np.asarray(m, dtype=np.complex128).reshape(-1, 2, 2)
    out = []
    for i, j in ((0, 0), (1, 0), (0, 1), (1, 1)):
        out += [np.ascontiguousarray(m[:, i, j].real), np.ascontiguousarray(m[:, i, j].imag)]
    return tuple(out)


def rows(m):
    return [(p, None) for p in real(m)]


# scaling (test_svd2.py:64-116) --------------------------------------------

def test_scale_known_shifts():
    res = svd2.compute_scale(real([[1, 0], [0, 1]]))
    assert res.shift[0] == 1021.0 and res.parts[0][0] == 2.0 ** 1021 and res.parts[1][0] == 0.0
    res = svd2.compute_scale(real([[DBL_MAX, DBL_MAX], [DBL_MAX, -DBL_MAX]]))
    assert res.shift[0] == -2.0 and res.parts[0][0] == DBL_MAX * 0.25
    assert (np.abs([p[0] for p in res.parts]) < 2.0 ** 1022).all()
    res = svd2.compute_scale(real([[0.0, 0.0], [0.0, 0.0]]))
    assert res.shift[0] == DBL_MAX and res.parts[0][0] == 0.0
    res = svd2.compute_scale(real([[TRUE_MIN, 0.0], [0.0, DBL_MAX]]))
    assert res.shift[0] == -2.0
    assert svd2.compute_scale(cplx([[3 + 4j, 0], [0, 0]])).shift[0] == 1019.0


def test_scale_bounds_and_roundtrip():
    rng = np.random.default_rng(21)
    vals = rng.integers(0, 2 ** 64, (4, 4096), dtype=np.uint64).view(np.float64)
    vals[~np.isfinite(vals)] = DBL_MAX
    assert (svd2.compute_scale(tuple(vals)).shift >= -2.0).all()
    rng = np.random.default_rng(22)
    parts = tuple(rng.standard_normal(512) * np.exp2(rng.integers(-900, 900, 512)) for _ in range(4))
    res = svd2.compute_scale(parts)
    for orig, scaled in zip(parts, res.parts):
        assert np.array_equal(bits(lanes.scalef(scaled, -res.shift)), bits(orig))


# norms, pivot, row sort (test_svd2.py:122-188) -----------------------------

def test_column_norms():
    m11, m21, m12, m22, n1, n2 = svd2.column_norms(*rows([[3, 0], [4, 2]]))
    assert (m11[0], m21[0], m12[0], m22[0], n1[0], n2[0]) == (3, 4, 0, 2, 5, 2)
    p = cplx([[3 + 4j, 0], [0, 1j]])
    m11, m21, m12, m22, n1, n2 = svd2.column_norms(*[(p[i], p[i + 1]) for i in range(0, 8, 2)])
    assert m11[0] == 5.0 and m22[0] == 1.0 and n1[0] == 5.0 and n2[0] == 1.0
    big = 2.0 ** 1021
    *_, n1, n2 = svd2.column_norms(*rows([[big, big], [big, big]]))
    want = np.sqrt(2.0) * big
    assert np.isfinite(n1[0]) and abs(n1[0] - want) < 4 * np.spacing(want)


def test_column_pivot_and_row_sort():
    e = rows([[1, 10], [0, 0]])
    r = svd2.column_norms(*e)
    (e11, e21, e12, e22), mags, n1, n2, swap = svd2.column_pivot(tuple(e), r[:4], r[4], r[5])
    assert swap[0] and e11[0][0] == 10.0 and e12[0][0] == 1.0 and n1[0] == 10.0 and n2[0] == 1.0
    e = rows([[2, 2], [0, 0]])
    r = svd2.column_norms(*e)
    (e11, *_), _, _, _, swap = svd2.column_pivot(tuple(e), r[:4], r[4], r[5])
    assert not swap[0] and e11[0][0] == 2.0                      # ties keep the order
    e = rows([[1, 0.5], [-3, 0.25]])
    r = svd2.column_norms(*e)
    piv, mags, *_ = svd2.column_pivot(tuple(e), r[:4], r[4], r[5])
    (e11, e21, e12, e22), mags2, swap = svd2.row_sort(piv, mags)
    assert swap[0] and (e11[0][0], e21[0][0], e12[0][0], e22[0][0]) == (-3.0, 1.0, 0.25, 0.5)
    assert mags2[0][0] == 3.0


# row phases, Givens, phase fix (test_svd2.py:194-267) ----------------------

def test_left_phase_reduce():
    e = [(a(-3.0), None), (a(4.0), None), (a(2.0), None), (a(-5.0), None)]
    b11, b21, f12, f22, ph1, ph2 = svd2.left_phase_reduce(*e, a(3.0), a(4.0))
    assert b11[0] == 3.0 and b21[0] == 4.0 and f12[0][0] == -2.0 and f22[0][0] == -5.0
    assert np.signbit(ph1[0][0]) and not np.signbit(ph2[0][0])
    p = cplx([[3 + 4j, 1 + 0j], [0j, 0j]])
    e = [(p[i], p[i + 1]) for i in range(0, 8, 2)]
    b11, b21, f12, f22, ph1, ph2 = svd2.left_phase_reduce(*e, a(5.0), a(0.0))
    assert ph1[0][0] == 0.6 and ph1[1][0] == 0.8 and f12[0][0] == 0.6 and f12[1][0] == -0.8
    assert ph2[0][0] == 1.0 and ph2[1][0] == 0.0


def test_givens_qr():
    tan, cos, r11, g12, g22 = svd2.givens_qr(a(4.0), a(3.0), (a(2.0), None), (a(-1.0), None), a(5.0))
    assert (tan[0], cos[0], r11[0], g12[0][0], g22[0][0]) == (-0.75, 0.8, 5.0, 1.0, -2.0)
    tan, cos, r11, g12, g22 = svd2.givens_qr(a(4.0), a(0.0), (a(7.0), None), (a(3.0), None), a(4.0))
    assert bits(tan)[0] == bits(a(-0.0))[0] and cos[0] == 1.0
    assert g12[0][0] == 7.0 and g22[0][0] == 3.0
    tan, cos, r11, *_ = svd2.givens_qr(a(0.0), a(0.0), (a(0.0), None), (a(0.0), None), a(0.0))
    assert bits(tan)[0] == bits(a(-0.0))[0] and cos[0] == 1.0 and r11[0] == 0.0


def test_phase_fix_r():
    r12, r22, dt, dh = svd2.phase_fix_r((a(1.0), None), (a(-2.0), None))
    assert r12[0] == 1.0 and r22[0] == 2.0 and not np.signbit(dt[0][0]) and np.signbit(dh[0][0])
    r12, r22, dt, dh = svd2.phase_fix_r((a(-3.0), None), (a(4.0), None))
    assert r12[0] == 3.0 and r22[0] == 4.0 and np.signbit(dt[0][0]) and np.signbit(dh[0][0])
    r12, r22, dt, dh = svd2.phase_fix_r((a(0.0), a(4.0)), (a(2.0), a(0.0)))
    assert r12[0] == 4.0 and dt[0][0] == 0.0 and dt[1][0] == -1.0
    assert r22[0] == 2.0 and dh[0][0] == 0.0 and dh[1][0] == -1.0


# triangle SVD (test_svd2.py:274-346) ----------------------------------------

def test_triangle_known_answers():
    t = svd2.triangular_svd(a(1.0), a(0.0), a(1.0))
    assert bits(t.left_tan)[0] == bits(a(-0.0))[0] and t.left_cos[0] == 1.0
    assert t.right_cos[0] == 1.0 and t.smax_scaled[0] == 1.0 and t.smin_scaled[0] == 1.0
    t = svd2.triangular_svd(a(2.0), a(1.0), a(1.0))
    assert abs(t.left_tan[0] - -0.2360679774997897) <= 2 * EPS
    assert abs(t.right_tan[0] - -0.6180339887498949) <= 2 * EPS
    assert abs(t.smax_scaled[0] - 2.288245611270737) <= 8 * EPS * 2.288245611270737
    assert abs(t.smin_scaled[0] - 0.8740320488976422) <= 8 * EPS * 0.8740320488976422
    t = svd2.triangular_svd(a(1.0), a(1.0), a(0.0))
    assert bits(t.left_tan)[0] == bits(a(-0.0))[0] and t.right_tan[0] == -1.0
    assert t.right_cos[0] == lanes.invsqrt_lane(a(2.0))[0] and t.smin_scaled[0] == 0.0
    assert abs(t.smax_scaled[0] - np.sqrt(2.0)) <= np.spacing(np.sqrt(2.0))
    t = svd2.triangular_svd(a(0.0), a(0.0), a(0.0))
    assert bits(t.left_tan)[0] == bits(a(-0.0))[0] and t.right_tan[0] == -0.0
    assert t.left_cos[0] == 1.0 and t.smax_scaled[0] == 0.0 and t.smin_scaled[0] == 0.0
    t = svd2.triangular_svd(a(1.0), a(2.0 ** -540), a(1.0))
    assert t.left_tan[0] == -1.0 and abs(t.right_tan[0]) <= np.sqrt(2.0) * (1 + 2 * EPS)
    assert np.isfinite(t.smax_scaled[0]) and t.smax_scaled[0] >= t.smin_scaled[0] >= 0.0


def test_triangle_invariants_random():
    rng = np.random.default_rng(23)
    n = 1 << 15
    r11 = np.exp2(rng.uniform(-500, 1021, n))
    radius = np.sqrt(rng.uniform(0, 1, n))
    angle = rng.uniform(0, np.pi / 2, n)
    r12, r22 = r11 * (radius * np.cos(angle)), r11 * (radius * np.sin(angle))
    t = svd2.triangular_svd(r11, r12, r22)
    assert (np.abs(t.left_tan) <= 1.0).all()
    assert (np.abs(t.right_tan) <= np.sqrt(2.0) * (1 + 2 * EPS)).all()
    assert (np.abs(t.right_tan) >= np.abs(t.left_tan)).all()
    assert (t.right_cos >= (1 / np.sqrt(3.0)) * (1 - 2 * EPS)).all()
    assert (t.smax_scaled >= t.smin_scaled).all() and (t.smin_scaled >= 0.0).all()
    assert (t.smax_scaled <= np.sqrt(3.0) * (1 + 4 * EPS) * r11).all()
    assert np.isfinite(t.smax_scaled).all()


# whole pipeline (test_svd2.py:353-440) ---------------------------------------

def _u(s, k):
    return np.array([[s.u11[0][k], s.u12[0][k]], [s.u21[0][k], s.u22[0][k]]])


def _v(s, k):
    return np.array([[s.v11[0][k], s.v12[0][k]], [s.v21[0][k], s.v22[0][k]]])


def test_pipeline_known_answers():
    s = svd2.svd2_lanes(real([[1, 0], [0, 1]]))
    assert s.shift[0] == 1021.0 and s.smax_scaled[0] == 2.0 ** 1021 and s.smin_scaled[0] == 2.0 ** 1021
    assert _u(s, 0).tolist() == [[1, 0], [0, 1]] and _v(s, 0).tolist() == [[1, 0], [0, 1]]
    s = svd2.svd2_lanes(real([[4, 2], [3, -1]]))
    assert s.shift[0] == 1019.0
    smax, smin, sh = svd2.backscale(s.smax_scaled, s.smin_scaled, s.shift, mode="safe")
    assert abs(smax[0] - 5.116672736016927) <= 1e-6 * 5.116672736016927
    assert abs(smin[0] - 1.954395075848548) <= 1e-6 * 1.954395075848548
    assert np.signbit(sh[0]) and sh[0] == 0.0
    u, v = _u(s, 0), _v(s, 0)
    assert abs(u[0, 0] - 0.8506508083520399) <= 1e-6 and abs(u[1, 0] - 0.5257311121191336) <= 1e-6
    assert abs(v[0, 0] - 0.9732489894677302) <= 1e-6 and abs(v[1, 0] - 0.22975292054736118) <= 1e-6
    assert np.abs(u @ np.diag([smax[0], smin[0]]) @ v.T - [[4, 2], [3, -1]]).max() <= 1e-13


def test_pipeline_swap_symmetries_bitwise():
    base = svd2.svd2_lanes(real([[4, 2], [3, -1]]))
    rs = svd2.svd2_lanes(real([[3, -1], [4, 2]]))
    cs = svd2.svd2_lanes(real([[2, 4], [-1, 3]]))
    for sw in (rs, cs):
        assert bits(sw.smax_scaled)[0] == bits(base.smax_scaled)[0]
    for x, y in (("u11", "u21"), ("u21", "u11"), ("u12", "u22"), ("u22", "u12")):
        assert bits(getattr(rs, x)[0])[0] == bits(getattr(base, y)[0])[0]
        assert bits(getattr(cs, x)[0])[0] == bits(getattr(base, x)[0])[0]
    for x, y in (("v11", "v21"), ("v21", "v11"), ("v12", "v22"), ("v22", "v12")):
        assert bits(getattr(cs, x)[0])[0] == bits(getattr(base, y)[0])[0]
        assert bits(getattr(rs, x)[0])[0] == bits(getattr(base, x)[0])[0]


def test_pipeline_complex_against_oracle_svd2():
    from paper_2005_07403_b200 import oracle_svd2
    rng = np.random.default_rng(24)
    mats = rng.standard_normal((256, 2, 2)) + 1j * rng.standard_normal((256, 2, 2))
    s = svd2.svd2_lanes(cplx(mats))
    ref = oracle_svd2(mats)
    smax = s.smax_scaled * np.exp2(-s.shift)
    assert (np.abs(smax - ref.smax.hi) <= 2.0 ** -45 * ref.smax.hi).all()


def test_lane_purity():
    """A lane's result does not depend on its neighbours (test_svd2.py:428-440)."""
    rng = np.random.default_rng(25)
    parts = tuple(rng.standard_normal(64) * np.exp2(rng.integers(-300, 300, 64)) for _ in range(4))
    whole = svd2.svd2_lanes(parts)
    for k in (0, 17, 63):
        one = svd2.svd2_lanes(tuple(p[k:k + 1] for p in parts))
        assert bits(one.smax_scaled)[0] == bits(whole.smax_scaled)[k]
        assert bits(one.u21[0])[0] == bits(whole.u21[0])[k]
