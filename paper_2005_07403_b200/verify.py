"""Batch quality metrics on the GPU (drop-in for lanesvd.verify.metrics).

``metrics(batch, out)`` runs the double-double verifier kernel
(csrc/b2s_verify.cu, C-ABI ``b2s_metrics``) over every genuine lane and
folds the per-block exact maxima on the host into the reference's
``Metrics`` record (verify.py:355-372): kappa, rho, delta, eta as mpmath
numbers carrying the full double-double value, and the count of lanes whose
stored singular values are non-finite.  Per-lane values are bit-identical to
the reference's, so the maxima are too; unlike the reference (~10^5
lanes/s/core) it covers a 2^30-lane batch in one pass.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib
from .layout import is_device_array

__all__ = ["Metrics", "metrics", "lane_metrics", "fold_partials", "DD", "OracleSvd",
           "oracle_svd2"]

_NPART = 17


@dataclass
class Metrics:
    """Worst-lane quality measures (verify.py:355-372)."""
    kappa: object
    rho: object
    delta: object
    eta: object
    rho_excluded_lanes: int = 0
    # exact double-double parts, for bit-level comparisons
    raw: dict = None


def _dev(x, device):
    import torch
    if is_device_array(x):
        return x.contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(device)


def _run(batch, out, lane_values):
    import torch
    n = batch.n
    if out.n != n:
        raise ValueError("batch and output sizes differ")
    device = batch.re.device if batch.on_device else (
        out.u_re.device if out.on_device else torch.device("cuda", torch.cuda.current_device()))
    cplx = batch.im is not None
    tr = lambda a: None if a is None else [_dev(a[t][:n], device) for t in range(4)]
    a_re, a_im = tr(batch.re), tr(batch.im)
    u_re, u_im = tr(out.u_re), tr(out.u_im)
    v_re, v_im = tr(out.v_re), tr(out.v_im)
    sv = [_dev(x[:n], device) for x in (out.smax, out.smin, out.shift)]
    props = torch.cuda.get_device_properties(device)
    blocks = max(1, min(props.multi_processor_count * 8, -(-n // 128)))
    partial = torch.empty((blocks, _NPART), dtype=torch.float64, device=device)
    lanes = [torch.empty(n, dtype=torch.float64, device=device) for _ in range(3)] \
        if lane_values else None
    P = lambda rows: (None, None) if rows is None else _lib.ptr_array([r.data_ptr() for r in rows])
    ar, k1 = P(a_re)
    ai, k2 = P(a_im)
    ur, k3 = P(u_re)
    ui, k4 = P(u_im)
    vr, k5 = P(v_re)
    vi, k6 = P(v_im)
    lp = [l.data_ptr() for l in lanes] if lanes else [None, None, None]
    with torch.cuda.device(device):
        rc = _metrics_call(n, ar, ai, ur, ui, vr, vi, sv, partial, blocks, lp, cplx, device)
    _lib.check(rc, "b2s_metrics")
    return partial.cpu().numpy(), lanes


def _metrics_call(n, ar, ai, ur, ui, vr, vi, sv, partial, blocks, lp, cplx, device):
    import torch
    return _lib.lib.b2s_metrics(n, ar, ai if cplx else None, ur, ui if cplx else None, vr,
                              vi if cplx else None, sv[0].data_ptr(), sv[1].data_ptr(),
                              sv[2].data_ptr(), partial.data_ptr(), blocks, *lp,
                              torch.cuda.current_stream(device).cuda_stream)


def fold_partials(p):
    """Exact lexicographic maxima over per-block partial records."""
    def dd_max(h, l):
        mh = np.max(h)
        return mh, np.max(l[h == mh]) if np.isfinite(mh) else mh
    rho = dd_max(p[:, 0], p[:, 1])
    delta = dd_max(p[:, 2], p[:, 3])
    eta = dd_max(p[:, 4], p[:, 5])
    d = p[:, 6]
    dmax = np.max(d)
    sel = d == dmax
    qhi = np.max(p[sel, 7])
    sel &= p[:, 7] == qhi
    qlo = np.max(p[sel, 8])
    return {"rho": rho, "delta": delta, "eta": eta, "kappa": (dmax, qhi, qlo),
            "kappa_inf": bool(np.max(p[:, 9]) > 0), "excluded": int(np.sum(p[:, 10])),
            "delta2": dd_max(p[:, 11], p[:, 12]), "eta2": dd_max(p[:, 13], p[:, 14]),
            "over_8eps_frobenius": int(np.sum(p[:, 15])), "over_8eps_2norm": int(np.sum(p[:, 16]))}


def metrics(batch, out):
    """Worst-lane quality measures of ``out`` against ``batch``
    (verify.py:395-477), computed on the GPU."""
    import mpmath
    p, _ = _run(batch, out, False)
    f = fold_partials(p)
    with mpmath.workprec(240):
        mp = lambda hl: mpmath.mpf(float(hl[0])) + mpmath.mpf(float(hl[1]))
        if f["kappa_inf"]:
            kappa = mpmath.mpf("inf")
        else:
            dmax, qhi, qlo = f["kappa"]
            kappa = (mpmath.mpf(float(qhi)) + mpmath.mpf(float(qlo))) * mpmath.power(2, int(dmax))
        return Metrics(kappa=kappa, rho=mp(f["rho"]), delta=mp(f["delta"]),
                       eta=mp(f["eta"]), rho_excluded_lanes=f["excluded"], raw=f)


def lane_metrics(batch, out):
    """Per-lane (rho, delta, eta) high parts as device tensors, plus the
    folded batch record."""
    p, lanes = _run(batch, out, True)
    return lanes, fold_partials(p)


# ---------------------------------------------------------------------------
# independent reference SVD (verify.py:222-352)
# ---------------------------------------------------------------------------

class DD(NamedTuple):
    """Double-double values (verify.py:42-45): hi + lo, |lo| <= ulp(hi)/2."""
    hi: np.ndarray
    lo: np.ndarray


@dataclass
class OracleSvd:
    """Reference factors in double-double, one lane per array slot
    (verify.py:222-252): ``smax``/``smin`` DD arrays; factor entries complex
    double-double pairs (DD re, DD im), imaginary parts exactly zero for real
    input."""
    smax: DD
    smin: DD
    u11: tuple
    u21: tuple
    u12: tuple
    u22: tuple
    v11: tuple
    v21: tuple
    v12: tuple
    v22: tuple

    def u_array(self, k):
        return _factor_array((self.u11, self.u12, self.u21, self.u22), k)

    def v_array(self, k):
        return _factor_array((self.v11, self.v12, self.v21, self.v22), k)


def _factor_array(entries, k):
    """Lane k's factor as a 2x2 complex128 matrix (entries in row-major
    order; each double-double part rounded to one double)."""
    z = np.empty(4, dtype=np.complex128)
    for j, (re, im) in enumerate(entries):
        z[j] = complex(float(re.hi[k]) + float(re.lo[k]), float(im.hi[k]) + float(im.lo[k]))
    return z.reshape(2, 2)


def oracle_svd2(matrices, device=None):
    """Closed-form reference SVD of 2x2 lanes in double-double
    (lanesvd.verify.oracle_svd2, verify.py:259-352), computed on the GPU by
    ``b2s_oracle_svd2`` with the reference's own double-double operation
    sequence -- every output word bit-identical.  Accepts one (2, 2) matrix
    or an (n, 2, 2) stack, real or complex; returns host arrays."""
    import torch
    a = np.asarray(matrices)
    if a.shape == (2, 2):
        a = a.reshape(1, 2, 2)
    if a.ndim != 3 or a.shape[1:] != (2, 2):
        raise ValueError("expected (n, 2, 2) matrices, got %r" % (a.shape,))
    cplx = bool(np.iscomplexobj(a))
    if cplx:
        a = a.astype(np.complex128, copy=False)
        parts_re, parts_im = a.real, a.imag
    else:
        parts_re, parts_im = a.astype(np.float64, copy=False), None
    n = a.shape[0]
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    # trains in column-major entry order: e11, e21, e12, e22 (layout.py:3-10)
    order = ((0, 0), (1, 0), (0, 1), (1, 1))
    up = lambda p: torch.from_numpy(np.ascontiguousarray(
        np.stack([p[:, i, j] for i, j in order]), dtype=np.float64)).to(device)
    tre = up(parts_re)
    tim = up(parts_im) if cplx else None
    out = torch.empty((36, max(n, 1)), dtype=torch.float64, device=device)
    ar, k1 = _lib.ptr_array([tre[t].data_ptr() for t in range(4)])
    ai, k2 = (None, None) if tim is None else _lib.ptr_array([tim[t].data_ptr() for t in range(4)])
    op, k3 = _lib.ptr_array([out[k].data_ptr() for k in range(36)])
    with torch.cuda.device(device):
        rc = _lib.lib.b2s_oracle_svd2(n, ar, ai, op, torch.cuda.current_stream(device).cuda_stream)
    _lib.check(rc, "b2s_oracle_svd2")
    h = out[:, :n].cpu().numpy()
    dd = lambda k: DD(h[k].copy(), h[k + 1].copy())
    cd = lambda k: (dd(4 + 4 * k), dd(6 + 4 * k))
    return OracleSvd(smax=dd(0), smin=dd(2), u11=cd(0), u21=cd(1), u12=cd(2), u22=cd(3),
                     v11=cd(4), v21=cd(5), v12=cd(6), v22=cd(7))
