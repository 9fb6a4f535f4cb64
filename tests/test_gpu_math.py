"""The engine's inline sqrt / reciprocal / division sequences vs IEEE.

The fast pipeline replaces the library's div.rn / sqrt.rn expansions with
inline seed + Newton sequences (csrc/b2s_lane.cuh) and range-checked call
sites (csrc/b2s_fast.cuh).  Here each is compared bit for bit with torch's
IEEE-correct CUDA operations over large random operand sets in (and at the
edges of) the ranges the pipeline feeds them.  Checked sites may decline
(write the hard marker) but must never return a wrong value.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2005_07403_b200 import _lib  # noqa: E402

DEV = torch.device("cuda", 0)
HARD = 0x7FF4DEADBEEF0000
N = 1 << 24


def probe(op, a, b=None):
    out = torch.empty_like(a)
    rc = _lib.lib.b2s_math_probe(op, a.numel(), a.data_ptr(),
                                 None if b is None else b.data_ptr(),
                                 out.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "b2s_math_probe")
    return out


def bits(t):
    return t.view(torch.int64)


def rand_mag(n, lo_exp, hi_exp, gen):
    """|x| = U[1,2) * 2^e, e uniform in [lo_exp, hi_exp] (float64, device)."""
    m = 1.0 + torch.rand(n, dtype=torch.float64, device=DEV, generator=gen)
    e = torch.randint(lo_exp, hi_exp + 1, (n,), device=DEV, generator=gen)
    return torch.ldexp(m, e.to(torch.float64))


def rand_bits(n, gen):
    x = torch.randint(-(1 << 62), 1 << 62, (n,), dtype=torch.int64, device=DEV, generator=gen)
    x = x * 2 + torch.randint(0, 2, (n,), dtype=torch.int64, device=DEV, generator=gen)
    return x.view(torch.float64)


def assert_same(got, ref, what):
    bad = (bits(got) != bits(ref)).nonzero()
    if bad.numel():
        k = bad[0].item()
        raise AssertionError("%s: %d mismatches, e.g. got %r ref %r" % (
            what, bad.numel(), got[k].item(), ref[k].item()))


@pytest.fixture
def gen():
    g = torch.Generator(device=DEV)
    g.manual_seed(1234)
    return g


def test_sqrt_full_range(gen):
    for lo, hi in ((-960, 1023), (0, 1), (-1, 2), (1020, 1023)):
        x = rand_mag(N, lo, hi, gen)
        assert_same(probe(1, x), torch.sqrt(x), "sqrt [2^%d, 2^%d]" % (lo, hi))
    # boundary operands: 1, 1 +- ulps, DBL_MAX, perfect squares
    x = torch.tensor([1.0, np.nextafter(1.0, 2), np.nextafter(1.0, 0), 4.0, 2.0,
                      1.7976931348623157e308, np.nextafter(4.0, 0), 9.0, 3.0],
                     dtype=torch.float64, device=DEV)
    assert_same(probe(1, x), torch.sqrt(x), "sqrt edges")


def test_reciprocal_and_invsqrt(gen):
    x = rand_mag(N, -1000, 1000, gen)
    assert_same(probe(2, x), 1.0 / x, "rcp")
    z = 1.0 + 2.0 * torch.rand(N, dtype=torch.float64, device=DEV, generator=gen)   # [1, 3]
    assert_same(probe(3, z), 1.0 / torch.sqrt(z), "invsqrt")


def test_raw_quotient_in_range(gen):
    b = rand_mag(N, -900, 1000, gen)
    a = rand_mag(N, -900, 1000, gen) * torch.where(
        torch.rand(N, device=DEV, generator=gen) < 0.5, -1.0, 1.0).to(torch.float64)
    q = probe(0, a, b)
    ref = a / b
    ok = (ref.abs() > 2.0 ** -1021) & (ref.abs() < 2.0 ** 1022)
    assert_same(q[ok], ref[ok], "quot_f")


def test_checked_division_never_wrong(gen):
    # 0 <= a <= b < 2^1024, including huge denominators and tiny numerators
    for lo, hi, spread in ((1019, 1023, 60), (-50, 50, 60), (1000, 1023, 2100), (-1022, 1022, 2100)):
        b = rand_mag(N, lo, hi, gen)
        a = b * torch.rand(N, dtype=torch.float64, device=DEV, generator=gen) * torch.ldexp(
            torch.ones(N, dtype=torch.float64, device=DEV),
            -torch.randint(0, spread, (N,), device=DEV, generator=gen).to(torch.float64))
        a[:1000] = 0.0
        q = probe(9, a, b)
        hard = bits(q) == HARD
        assert_same(q[~hard], (a / b)[~hard], "div_pos_big_f")
        if spread < 100:
            assert hard.float().mean().item() < 1e-3


def test_normalised_division_full_range(gen):
    """div_den: exact for every normal/zero numerator and normal denominator,
    including subnormal and overflowing quotients; declines only subnormal
    operands."""
    sgn = lambda: torch.where(torch.rand(N, device=DEV, generator=gen) < 0.5, -1.0, 1.0).to(torch.float64)
    for (la, ha), (lb, hb) in (((-1022, 1023), (-1022, 1023)), ((-1022, -900), (900, 1023)),
                               ((1000, 1023), (-1022, -1000)), ((-60, 60), (-60, 60))):
        a = rand_mag(N, la, ha, gen) * sgn()
        b = rand_mag(N, lb, hb, gen) * sgn()
        a[:1000] = 0.0
        a[1000:2000] = -0.0
        q = probe(6, a, b)
        hard = bits(q) == HARD
        assert not hard.any()
        assert_same(q, a / b, "div_den [%d,%d]/[%d,%d]" % (la, ha, lb, hb))
    # exact ties on the subnormal grid: d = D 2^1000 with a short mantissa D,
    # a = D (2k+1) 2^-75 exactly, so a / d = (2k+1) 2^-1075 (a midpoint)
    D = 1.0 + torch.randint(0, 1024, (N,), device=DEV, generator=gen).to(torch.float64) / 1024.0
    k = torch.randint(0, 64, (N,), device=DEV, generator=gen).to(torch.float64)
    d = D * 2.0 ** 1000
    a = D * (2 * k + 1) * 2.0 ** -75
    q = probe(6, a, d)
    assert_same(q, a / d, "subnormal ties")
    # subnormal operands are normalised exactly
    a = rand_mag(N, -1074, -1023, gen) * sgn()
    b = rand_mag(N, -1074, 1023, gen) * sgn()
    q = probe(6, a, b)
    assert_same(q, a / b, "div_den subnormal operands")
    assert_same(probe(6, b, a), b / a, "div_den subnormal denominators")
    # zero denominators are declined
    z = torch.zeros(4, dtype=torch.float64, device=DEV)
    assert (bits(probe(6, a[:4], z)) == HARD).all()


@pytest.mark.parametrize("op", [10, 11, 12, 13])
def test_normalised_division_streaming_variant(gen, op):
    """div_den as the streaming kernels run it: selects instead of per-lane
    branches, subnormal quotients rounded by the warp-uniform FP64 sequence
    (op 10), the integer re-rounding call (op 11) or its inline select form
    (op 12, subnormal_quot_sel; op 13 the same under a warp-uniform branch).
    Exact for every normal /
    zero numerator over a normal denominator; declines subnormal operands."""
    sgn = lambda: torch.where(torch.rand(N, device=DEV, generator=gen) < 0.5, -1.0, 1.0).to(torch.float64)
    for (la, ha), (lb, hb) in (((-1022, 1023), (-1022, 1023)), ((-1022, -900), (900, 1023)),
                               ((-1022, -1000), (0, 80)), ((-200, 0), (850, 1023)),
                               ((1000, 1023), (-1022, -1000)), ((-60, 60), (-60, 60))):
        a = rand_mag(N, la, ha, gen) * sgn()
        b = rand_mag(N, lb, hb, gen) * sgn()
        a[:1000] = 0.0
        a[1000:2000] = -0.0
        q = probe(op, a, b)
        assert not (bits(q) == HARD).any()
        assert_same(q, a / b, "streaming div_den [%d,%d]/[%d,%d]" % (la, ha, lb, hb))
    # exact midpoints of the subnormal grid and their neighbours: a / d =
    # (2k+1) 2^-s exactly, s spanning every subnormal rounding position
    D = 1.0 + torch.randint(0, 1024, (N,), device=DEV, generator=gen).to(torch.float64) / 1024.0
    k = torch.randint(0, 1 << 20, (N,), device=DEV, generator=gen).to(torch.float64)
    s = torch.randint(1023, 1080, (N,), device=DEV, generator=gen)
    d = D * 2.0 ** 1000
    for nudge in (0, 1, -1):
        a = D * (2 * k + 1)
        a = torch.ldexp(a, (1000 - s).to(torch.float64))
        a = a.view(torch.int64).add(nudge).view(torch.float64)    # one ulp off the midpoint
        a = a * sgn()
        ok = a != 0
        q = probe(op, a[ok], d[ok])
        assert_same(q, a[ok] / d[ok], "streaming div_den ties nudge=%d" % nudge)
    # subnormal operands are declined, never wrong
    a = rand_mag(N, -1074, -1023, gen)
    b = rand_mag(N, 0, 10, gen)
    q = probe(op, a, b)
    assert (bits(q) == HARD).all()
    q = probe(op, b, a)
    assert (bits(q) == HARD).all()


def test_hypot_never_wrong(gen):
    import oracle
    for lo, hi in ((1015, 1022), (-1074, 1022), (-30, 30)):
        x = rand_mag(N, lo, hi, gen)
        y = rand_mag(N, lo, hi, gen)
        y[:4096] = 0.0
        got = probe(4, x, y)
        hard = (bits(got) == HARD).cpu().numpy()
        ref = oracle.hypot_vec(x.cpu().numpy(), y.cpu().numpy())
        g = got.cpu().numpy()
        assert (g[~hard].view(np.uint64) == ref[~hard].view(np.uint64)).all(), (lo, hi)
        if hi - lo < 100:
            assert hard.mean() < 1e-3


def test_phase_never_wrong(gen):
    import oracle
    sgn = lambda n: torch.where(torch.rand(n, device=DEV, generator=gen) < 0.5, -1.0, 1.0).to(torch.float64)
    for (lx, hx), (ly, hy) in (((-1074, 1022), (-60, 1022)), ((1000, 1022), (1000, 1022)), ((-20, 20), (-20, 20))):
        x = rand_mag(N, lx, hx, gen) * sgn(N)
        y = rand_mag(N, ly, hy, gen) * sgn(N)
        x[:100] = 0.0
        y[50:150] = -0.0
        c = probe(7, x, y).cpu().numpy()
        s = probe(8, x, y).cpu().numpy()
        rc, rs = oracle.phase_vec(x.cpu().numpy(), y.cpu().numpy())
        for got, ref, nm in ((c, rc, "cos"), (s, rs, "sin")):
            hard = got.view(np.uint64) == HARD
            assert (got[~hard].view(np.uint64) == ref[~hard].view(np.uint64)).all(), nm
            if hx - lx < 100:
                assert hard.mean() < 1e-3, nm


def test_scale_up_exact(gen):
    x = rand_bits(N, gen)
    x = torch.where(torch.isfinite(x), x, torch.zeros_like(x))
    s = torch.randint(-2, 2096, (N,), device=DEV, generator=gen).to(torch.float64)
    got = probe(5, x, s).cpu().numpy()
    xs, ss = x.cpu().numpy(), s.cpu().numpy().astype(np.int64)
    with np.errstate(over="ignore"):
        ref = np.ldexp(xs, ss)       # C ldexp: one correct rounding
    keep = np.isfinite(ref) & (np.abs(ref) <= 2.0 ** 1022)
    assert (got[keep].view(np.uint64) == ref[keep].view(np.uint64)).all()
