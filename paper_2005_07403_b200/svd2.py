"""Lane-level entry points of the GPU pipeline (drop-in for lanesvd.svd2).

``svd2_lanes`` and ``backscale`` keep the reference signatures
(svd2.py:521-570, 481-514) but run the fused sm_100a kernels through the
C-ABI.  Trains may be host NumPy arrays (staged through HBM and returned as
NumPy) or CUDA tensors (processed in place on their device, results left in
HBM).  The batch path fuses every phase in registers; its intermediate values are
exported by ``with_states=True`` as the reference's (Svd2, ScaleResult,
UrvState, TriangleSvd) tuple.  The phases also exist one at a time, with the
reference's signatures (compute_scale ... assemble_uv_sine), each one device
kernel over the same exact lane arithmetic (``b2s_svd2_phase``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .layout import is_device_array

__all__ = ["HEADROOM_EXP", "SQRT_DBL_MAX", "Svd2", "ScaleResult", "UrvState",
           "TriangleSvd", "dump_trains", "svd2_lanes", "backscale", "launch_device",
           "compute_scale", "column_norms", "column_pivot", "row_sort",
           "left_phase_reduce", "givens_qr", "phase_fix_r", "triangular_svd",
           "assemble_uv", "assemble_uv_sine"]

HEADROOM_EXP = 1021.0                  # svd2.py:52-56
SQRT_DBL_MAX = 1.34078079299425956e+154  # svd2.py:58-59

# driver.py:193-216 state-train order (B2S_FLAG_STATES), then the rest of the
# with_states tuple (B2S_FLAG_STATES_FULL): triangle sec2/cos, scaled parts
EXTRA_STATE_NAMES = ("left_sec2", "left_cos", "right_sec2", "right_cos")
STATE_NAMES_REAL = ("shift", "swap_cols", "swap_rows", "row_phase1",
                    "row_phase2", "r12_phase", "r22_phase", "givens_tan",
                    "givens_cos", "r11", "r12", "r22", "left_tan",
                    "right_tan", "smax_scaled", "smin_scaled")
STATE_NAMES_COMPLEX = ("shift", "swap_cols", "swap_rows",
                       "row_phase1_re", "row_phase1_im",
                       "row_phase2_re", "row_phase2_im",
                       "r12_phase_re", "r12_phase_im",
                       "r22_phase_re", "r22_phase_im", "givens_tan",
                       "givens_cos", "r11", "r12", "r22", "left_tan",
                       "right_tan", "smax_scaled", "smin_scaled")


@dataclass
class Svd2:
    """Assembled factors (svd2.py:108-127): U/V entries as (re, im) pairs in
    column-major entry order (im None for real lanes), scaled singular
    values and the shift."""
    u11: tuple
    u21: tuple
    u12: tuple
    u22: tuple
    v11: tuple
    v21: tuple
    v12: tuple
    v22: tuple
    smax_scaled: object
    smin_scaled: object
    shift: object


@dataclass
class ScaleResult:
    """svd2.py:61-65: exactly scaled component trains (input order) and the
    per-lane exponent s."""
    shift: object
    parts: tuple


@dataclass
class UrvState:
    """svd2.py:68-87: the unitary reduction to a non-negative triangle.
    Phases are (re, im) pairs (im None for real lanes)."""
    swap_cols: object
    swap_rows: object
    row_phase1: tuple
    row_phase2: tuple
    givens_tan: object
    givens_cos: object
    r12_phase: tuple
    r22_phase: tuple
    r11: object
    r12: object
    r22: object


@dataclass
class TriangleSvd:
    """svd2.py:90-105: closed-form SVD of the triangle."""
    left_tan: object
    left_sec2: object
    left_cos: object
    right_tan: object
    right_sec2: object
    right_cos: object
    smax_scaled: object
    smin_scaled: object


def dump_trains(scale, urv, tri):
    """The driver._dump_states train order (driver.py:193-216) of a
    with_states tuple: shift, swaps as 0.0/1.0, the four phases (re then im
    for complex lanes), Givens tan/cos, r11, r12, r22, the two tangents and
    the scaled singular values."""
    f = lambda m: (m.astype(np.float64) if isinstance(m, np.ndarray) else m.double())
    trains = [scale.shift, f(urv.swap_cols), f(urv.swap_rows)]
    for ph in (urv.row_phase1, urv.row_phase2, urv.r12_phase, urv.r22_phase):
        trains.append(ph[0])
        if ph[1] is not None:
            trains.append(ph[1])
    return trains + [urv.givens_tan, urv.givens_cos, urv.r11, urv.r12, urv.r22,
                     tri.left_tan, tri.right_tan, tri.smax_scaled, tri.smin_scaled]


def _stream_of(t):
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def _addr(t):
    return t.data_ptr()


def check_device_trains(trains, n, device, what):
    """Every train a float64 CUDA vector on ``device`` with at least ``n``
    unit-stride elements -- the C-ABI reads and writes raw pointers, so a
    float32, strided, short or foreign-device tensor would be an
    out-of-bounds access, not an error, without this check."""
    import torch
    for k, t in enumerate(trains):
        name = "%s[%d]" % (what, k)
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError("%s must be a CUDA tensor" % name)
        if t.dtype != torch.float64:
            raise ValueError("%s must be float64, got %s" % (name, t.dtype))
        if t.dim() != 1 or t.shape[0] < n:
            raise ValueError("%s must be a vector of >= %d lanes, got shape %s"
                             % (name, n, tuple(t.shape)))
        if n > 1 and t.stride(0) != 1:
            raise ValueError("%s must have unit stride" % name)
        if t.device != device:
            raise ValueError("%s is on %s, expected %s" % (name, t.device, device))


def launch_device(n, in_re, in_im, out, mode, flags=0, states=None,
                  stream=None):
    """Run the device C-ABI on CUDA tensors.

    in_re/in_im: sequences of 4 device trains (in_im None for real);
    out: dict with u_re, u_im, v_re, v_im (sequences of 4 trains) and smax,
    smin, shift trains; states: sequence of state trains or None.  Every
    train is validated (float64, unit stride, >= n lanes, one device).
    Launches asynchronously on ``stream`` (default: torch's current stream
    of the trains' device), with that device current."""
    import torch
    n = int(n)
    device = in_re[0].device if isinstance(in_re[0], torch.Tensor) else None
    cplx = in_im is not None
    if (out.get("u_im") is not None) != cplx or (out.get("v_im") is not None) != cplx:
        raise ValueError("output trains do not match the field")
    groups = [("in_re", in_re), ("u_re", out["u_re"]), ("v_re", out["v_re"]),
              ("smax/smin/shift", [out["smax"], out["smin"], out["shift"]])]
    if cplx:
        groups += [("in_im", in_im), ("u_im", out["u_im"]), ("v_im", out["v_im"])]
    if states is not None:
        groups.append(("states", states))
    base = len(STATE_NAMES_COMPLEX if cplx else STATE_NAMES_REAL)
    full = base + len(EXTRA_STATE_NAMES) + (8 if cplx else 4)
    want = {"smax/smin/shift": 3,
            "states": full if flags & _lib.FLAG_STATES_FULL else base}
    for what, trains in groups:
        if len(trains) != want.get(what, 4):
            raise ValueError("%s: expected %d trains, got %d"
                             % (what, want.get(what, 4), len(trains)))
        check_device_trains(trains, n, device, what)
    with torch.cuda.device(device):
        _launch(n, in_re, in_im, out, mode, flags, states,
                _stream_of(in_re[0]) if stream is None else stream)


def _launch(n, in_re, in_im, out, mode, flags, states, stream):
    a, _k1 = _lib.ptr_array([_addr(x) for x in in_re])
    u, _k2 = _lib.ptr_array([_addr(x) for x in out["u_re"]])
    v, _k3 = _lib.ptr_array([_addr(x) for x in out["v_re"]])
    st, _k4 = (None, None)
    if states is not None:
        st, _k4 = _lib.ptr_array([_addr(x) for x in states])
        flags |= _lib.FLAG_STATES
    if in_im is None:
        rc = _lib.lib.b2s_svd2_real(
            int(n), a, u, v, _addr(out["smax"]), _addr(out["smin"]),
            _addr(out["shift"]), mode, flags, st, stream)
        _lib.check(rc, "b2s_svd2_real")
        return
    ai, _k5 = _lib.ptr_array([_addr(x) for x in in_im])
    ui, _k6 = _lib.ptr_array([_addr(x) for x in out["u_im"]])
    vi, _k7 = _lib.ptr_array([_addr(x) for x in out["v_im"]])
    rc = _lib.lib.b2s_svd2_complex(
        int(n), a, ai, u, ui, v, vi, _addr(out["smax"]), _addr(out["smin"]),
        _addr(out["shift"]), mode, flags, st, stream)
    _lib.check(rc, "b2s_svd2_complex")


def _to_device(x, device):
    import torch
    if is_device_array(x):
        return x.to(device=device, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(device)


def svd2_lanes(parts, sine_form=False, with_states=False, device=None):
    """Full pipeline on component trains (svd2.py:521-570).

    parts: 4 trains (e11, e21, e12, e22) for real lanes or 8 with re/im
    interleaved per entry.  Returns ``Svd2``, or with ``with_states`` the
    reference's ``(Svd2, ScaleResult, UrvState, TriangleSvd)``; host inputs
    give host (NumPy) results, device inputs device tensors."""
    import torch
    if len(parts) not in (4, 8):
        raise ValueError("expected 4 or 8 component trains, got %d"
                         % len(parts))
    host = not is_device_array(parts[0])
    if device is None:
        device = parts[0].device if not host else torch.device(
            "cuda", torch.cuda.current_device())
    device = torch.device(device)
    dev_parts = [_to_device(p, device) for p in parts]
    n = int(dev_parts[0].shape[0])
    for p in dev_parts:
        if p.shape != (n,):
            raise ValueError("component trains must be equal-length vectors")
    _lib.assert_device_fp_env(device.index or 0)
    cplx = len(parts) == 8
    in_re = dev_parts[0::2] if cplx else dev_parts
    in_im = dev_parts[1::2] if cplx else None
    E = lambda: torch.empty(n, dtype=torch.float64, device=device)
    out = {"u_re": [E() for _ in range(4)], "v_re": [E() for _ in range(4)],
           "u_im": [E() for _ in range(4)] if cplx else None,
           "v_im": [E() for _ in range(4)] if cplx else None,
           "smax": E(), "smin": E(), "shift": E()}
    names = (STATE_NAMES_COMPLEX if cplx else STATE_NAMES_REAL) + EXTRA_STATE_NAMES
    states = [E() for _ in range(len(names) + len(parts))] if with_states else None
    flags = _lib.FLAG_SINE_FORM if sine_form else 0
    if with_states:
        flags |= _lib.FLAG_STATES_FULL
    launch_device(n, in_re, in_im, out, 0, flags, states)
    fin = (lambda t: t.cpu().numpy()) if host else (lambda t: t)
    pair = lambda k: (fin(out["u_re"][k]), fin(out["u_im"][k]) if cplx else None)
    vpair = lambda k: (fin(out["v_re"][k]), fin(out["v_im"][k]) if cplx else None)
    svd = Svd2(u11=pair(0), u21=pair(1), u12=pair(2), u22=pair(3),
               v11=vpair(0), v21=vpair(1), v12=vpair(2), v22=vpair(3),
               smax_scaled=fin(out["smax"]), smin_scaled=fin(out["smin"]),
               shift=fin(out["shift"]))
    if not with_states:
        return svd
    st = dict(zip(names, [fin(x) for x in states[:len(names)]]))
    scaled = tuple(fin(x) for x in states[len(names):])
    ph = lambda k: (st[k + "_re"], st[k + "_im"]) if cplx else (st[k], None)
    mask = lambda x: (x != 0.0)
    scale = ScaleResult(shift=st["shift"], parts=scaled)
    urv = UrvState(swap_cols=mask(st["swap_cols"]), swap_rows=mask(st["swap_rows"]),
                   row_phase1=ph("row_phase1"), row_phase2=ph("row_phase2"),
                   givens_tan=st["givens_tan"], givens_cos=st["givens_cos"],
                   r12_phase=ph("r12_phase"), r22_phase=ph("r22_phase"),
                   r11=st["r11"], r12=st["r12"], r22=st["r22"])
    tri = TriangleSvd(left_tan=st["left_tan"], left_sec2=st["left_sec2"],
                      left_cos=st["left_cos"], right_tan=st["right_tan"],
                      right_sec2=st["right_sec2"], right_cos=st["right_cos"],
                      smax_scaled=st["smax_scaled"], smin_scaled=st["smin_scaled"])
    return svd, scale, urv, tri


def backscale(smax_scaled, smin_scaled, shift, mode="safe"):
    """Divide the shift back out of the singular values (svd2.py:481-514),
    on the GPU.  Lanes rescaled get shift -0.0; "safe" refuses lanes whose
    values would overflow or leave the normal range."""
    import torch
    if mode not in _lib.BACKSCALE:
        raise ValueError("unknown backscale mode %r" % (mode,))
    host = not is_device_array(smax_scaled)
    device = (smax_scaled.device if not host
              else torch.device("cuda", torch.cuda.current_device()))
    ins = [_to_device(np.atleast_1d(x) if host else x, device).reshape(-1)
           for x in (smax_scaled, smin_scaled, shift)]
    n = int(ins[0].numel())
    if any(int(x.numel()) != n for x in ins):
        raise ValueError("smax, smin and shift must have the same length")
    outs = [torch.empty(n, dtype=torch.float64, device=device)
            for _ in range(3)]
    with torch.cuda.device(device):
        rc = _lib.lib.b2s_backscale(n, *[_addr(x) for x in ins],
                                    _lib.BACKSCALE[mode],
                                    *[_addr(x) for x in outs], _stream_of(ins[0]))
    _lib.check(rc, "b2s_backscale")
    if host:
        return tuple(o.cpu().numpy() for o in outs)
    return tuple(outs)


# ---------------------------------------------------------------------------
# The pipeline's phases one at a time (svd2.py:134-474): the reference's
# svd2 module API over b2s_svd2_phase.  Values are host NumPy arrays or
# device tensors (results come back where the inputs live); complex values
# are (re, im) pairs, real ones (x, None) as in the reference.
# ---------------------------------------------------------------------------

_PHASE = {"compute_scale": 0, "column_norms": 1, "column_pivot": 2, "row_sort": 3,
          "left_phase_reduce": 4, "givens_qr": 5, "phase_fix_r": 6,
          "triangular_svd": 7, "assemble_uv": 8}


def _phase(name, cplx, ins, n_out, sine=False, finite=False):
    """Run one phase kernel on the trains `ins`; returns `n_out` trains."""
    import torch
    host = not any(is_device_array(x) for x in ins)
    dev = next((x.device for x in ins if is_device_array(x)), None)
    if dev is None:
        dev = torch.device("cuda", torch.cuda.current_device())

    def up(x):
        if is_device_array(x):
            return x.to(device=dev, dtype=torch.float64).reshape(-1).contiguous()
        a = np.asarray(x)
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).to(dev)
    t = [up(x) for x in ins]
    n = int(t[0].numel())
    if any(int(x.numel()) != n for x in t):
        raise ValueError("%s: trains must be equal-length vectors" % name)
    if finite and not all(bool(torch.isfinite(x).all()) for x in t):
        raise ValueError("%s: non-finite component" % name)
    _lib.assert_device_fp_env(dev.index or 0)
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(n_out)]
    if n == 0:                                   # nothing to launch (empty tensors have no storage)
        return [x.cpu().numpy() for x in outs] if host else outs
    pi, _k1 = _lib.ptr_array([x.data_ptr() for x in t])
    po, _k2 = _lib.ptr_array([x.data_ptr() for x in outs])
    with torch.cuda.device(dev):
        rc = _lib.lib.b2s_svd2_phase(_PHASE[name], int(cplx), int(sine), n, len(t), pi,
                                     len(outs), po, torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(rc, "b2s_svd2_phase(%s)" % name)
    if host:
        return [x.cpu().numpy() for x in outs]
    return outs


def _flat(pairs):
    """(re, im|None) pairs -> trains, and whether they are complex."""
    cplx = pairs[0][1] is not None
    if any((p[1] is not None) != cplx for p in pairs):
        raise ValueError("mixed real and complex values")
    return [x for p in pairs for x in ((p[0], p[1]) if cplx else (p[0],))], cplx


def _pairs(trains, cplx, count):
    k = 2 if cplx else 1
    return tuple((trains[k * j], trains[k * j + 1] if cplx else None) for j in range(count))


def _mask(x):
    return x != 0.0


def compute_scale(parts):
    """Joint exact power-of-two scaling (svd2.py:134-160) of 4 real or 8
    complex component trains; finite components (as the batch path
    requires).  Returns ``ScaleResult``."""
    if len(parts) not in (4, 8):
        raise ValueError("expected 4 or 8 component trains, got %d" % len(parts))
    out = _phase("compute_scale", len(parts) == 8, list(parts), 1 + len(parts), finite=True)
    return ScaleResult(shift=out[0], parts=tuple(out[1:]))


def column_norms(e11, e21, e12, e22):
    """Entry magnitudes and column norms (svd2.py:167-182):
    ``(m11, m21, m12, m22, norm1, norm2)``."""
    tr, cplx = _flat((e11, e21, e12, e22))
    return tuple(_phase("column_norms", cplx, tr, 6))


def column_pivot(entries, mags, norm1, norm2):
    """Exchange columns where norm1 < norm2 (svd2.py:193-208): returns
    ``(entries, mags, n1, n2, swap)``."""
    tr, cplx = _flat(entries)
    k = len(tr)
    out = _phase("column_pivot", cplx, tr + list(mags) + [norm1, norm2], k + 7)
    return (_pairs(out, cplx, 4), tuple(out[k:k + 4]), out[k + 4], out[k + 5],
            _mask(out[k + 6]))


def row_sort(entries, mags):
    """Exchange rows where m11 < m21 (svd2.py:211-224): returns
    ``(entries, mags, swap)``."""
    tr, cplx = _flat(entries)
    k = len(tr)
    out = _phase("row_sort", cplx, tr + list(mags), k + 5)
    return _pairs(out, cplx, 4), tuple(out[k:k + 4]), _mask(out[k + 4])


def left_phase_reduce(e11, e21, e12, e22, m11, m21):
    """Row phases of the pivot column (svd2.py:227-250): returns
    ``(b11, b21, f12, f22, phase1, phase2)``."""
    tr, cplx = _flat((e11, e21, e12, e22))
    out = _phase("left_phase_reduce", cplx, tr + [m11, m21], 2 + len(tr))
    f12, f22, ph1, ph2 = _pairs(out[2:], cplx, 4)
    return out[0], out[1], f12, f22, ph1, ph2


def givens_qr(b11, b21, f12, f22, norm1):
    """One rotation annihilating the subdiagonal (svd2.py:253-276):
    returns ``(tan, cos, r11, g12, g22)``."""
    tr, cplx = _flat((f12, f22))
    out = _phase("givens_qr", cplx, [b11, b21] + tr + [norm1], 3 + len(tr))
    g12, g22 = _pairs(out[3:], cplx, 2)
    return out[0], out[1], out[2], g12, g22


def phase_fix_r(g12, g22):
    """Strip the phases of the rotated column 2 (svd2.py:279-299): returns
    ``(r12, r22, r12_phase, r22_phase)``."""
    tr, cplx = _flat((g12, g22))
    out = _phase("phase_fix_r", cplx, tr, 2 + len(tr))
    dt, dh = _pairs(out[2:], cplx, 2)
    return out[0], out[1], dt, dh


def triangular_svd(r11, r12, r22):
    """Closed-form SVD of the non-negative triangle (svd2.py:306-343)."""
    out = _phase("triangular_svd", False, [r11, r12, r22], 8)
    return TriangleSvd(*out)


def _assemble(urv, tri, shift, sine):
    tr, cplx = _flat((urv.row_phase1, urv.row_phase2))
    ph = tr
    dtr, _ = _flat((urv.r12_phase, urv.r22_phase))
    f = lambda m: (m.astype(np.float64) if isinstance(m, np.ndarray) else
                   m.double() if hasattr(m, "double") else np.asarray(m, dtype=np.float64))
    ins = ([f(urv.swap_cols), f(urv.swap_rows)] + ph + [urv.givens_tan, urv.givens_cos] + dtr +
           [urv.r11, urv.r12, urv.r22, tri.left_tan, tri.left_sec2, tri.left_cos, tri.right_tan,
            tri.right_sec2, tri.right_cos, tri.smax_scaled, tri.smin_scaled, shift])
    k = 2 if cplx else 1
    out = _phase("assemble_uv", cplx, ins, 8 * k + 3, sine=sine)
    u = _pairs(out[:4 * k], cplx, 4)
    v = _pairs(out[4 * k:8 * k], cplx, 4)
    return Svd2(u11=u[0], u21=u[1], u12=u[2], u22=u[3], v11=v[0], v21=v[1], v12=v[2],
                v22=v[3], smax_scaled=out[8 * k], smin_scaled=out[8 * k + 1],
                shift=out[8 * k + 2])


def assemble_uv(urv, tri, shift):
    """U and V from the reduction and the triangle SVD, tangent form
    (svd2.py:350-424)."""
    return _assemble(urv, tri, shift, False)


def assemble_uv_sine(urv, tri, shift):
    """The same through explicit sines (svd2.py:427-474)."""
    return _assemble(urv, tri, shift, True)
