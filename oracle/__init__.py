"""CPU oracle for the batched 2x2 SVD -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/_build/liboracle.so`` (built from
``svd2_oracle.c`` by ``oracle/Makefile``), a scalar C restatement of the
reference ``lanesvd`` pipeline (svd2.py:134-570, lanes.py:102-259).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module.  The product package never does.

Parity pin: checked bit for bit against outputs of the reference itself
(``tests/golden/``, produced by ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

MODES = {"none": 0, "safe": 1, "unconditional": 2}

_P = ctypes.POINTER(ctypes.c_double)
_PP = ctypes.POINTER(_P)


def build():
    """Compile the oracle (idempotent; make decides)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        i64, c_int = ctypes.c_int64, ctypes.c_int
        L.oracle_svd2_real.argtypes = [i64, _PP, _PP, _PP, _P, _P, _P,
                                       c_int, c_int, c_int, _PP]
        L.oracle_svd2_complex.argtypes = [i64, _PP, _PP, _PP, _PP, _PP, _PP,
                                          _P, _P, _P, c_int, c_int, c_int,
                                          _PP]
        for name in ("oracle_getexp", "oracle_invsqrt"):
            getattr(L, name).argtypes = [ctypes.c_double]
            getattr(L, name).restype = ctypes.c_double
        for name in ("oracle_scalef", "oracle_hypot"):
            getattr(L, name).argtypes = [ctypes.c_double, ctypes.c_double]
            getattr(L, name).restype = ctypes.c_double
        L.oracle_backscale.argtypes = [i64, _P, _P, _P, c_int, _P, _P, _P]
        L.oracle_hypot_vec.argtypes = [i64, _P, _P, _P]
        L.oracle_phase_vec.argtypes = [i64, _P, _P, _P, _P]
        _lib = L
    return _lib


def _ptr(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_P)


def _ptrs(rows):
    arr = (_P * len(rows))(*[_ptr(r) for r in rows])
    return ctypes.cast(arr, _PP), arr


class OracleOut:
    """Same fields as ``lanesvd.layout.SvdBatchOut`` (layout.py:106-130)."""

    def __init__(self, n, cplx):
        self.n = n
        mk = lambda: np.zeros((4, n), dtype=np.float64)
        self.u_re, self.v_re = mk(), mk()
        self.u_im = mk() if cplx else None
        self.v_im = mk() if cplx else None
        self.smax = np.zeros(n)
        self.smin = np.zeros(n)
        self.shift = np.zeros(n)
        self.states = None

    def trains(self):
        """Named output trains in a fixed order."""
        out = {"u_re": self.u_re, "v_re": self.v_re, "smax": self.smax,
               "smin": self.smin, "shift": self.shift}
        if self.u_im is not None:
            out["u_im"] = self.u_im
            out["v_im"] = self.v_im
        return out


def svd2(re, im=None, backscale_mode="none", sine_form=False, threads=None,
         with_states=False):
    """Decompose (4, n) trains (plus (4, n) imaginary trains if complex)."""
    re = np.ascontiguousarray(re, dtype=np.float64)
    if re.ndim != 2 or re.shape[0] != 4:
        raise ValueError("expected (4, n) trains")
    n = re.shape[1]
    cplx = im is not None
    if cplx:
        im = np.ascontiguousarray(im, dtype=np.float64)
        if im.shape != re.shape:
            raise ValueError("re/im train shapes differ")
    if threads is None:
        threads = os.cpu_count() or 1
    out = OracleOut(n, cplx)
    keep = []
    a_re, k1 = _ptrs([re[t] for t in range(4)])
    keep.append(k1)
    u_re, k = _ptrs([out.u_re[t] for t in range(4)]); keep.append(k)
    v_re, k = _ptrs([out.v_re[t] for t in range(4)]); keep.append(k)
    st = None
    if with_states:
        out.states = np.zeros((20 if cplx else 16, n))
        st, k = _ptrs([out.states[t] for t in range(out.states.shape[0])])
        keep.append(k)
    mode = MODES[backscale_mode]
    if not cplx:
        rc = lib().oracle_svd2_real(n, a_re, u_re, v_re, _ptr(out.smax),
                                    _ptr(out.smin), _ptr(out.shift), mode,
                                    int(sine_form), threads, st)
    else:
        a_im, k = _ptrs([im[t] for t in range(4)]); keep.append(k)
        u_im, k = _ptrs([out.u_im[t] for t in range(4)]); keep.append(k)
        v_im, k = _ptrs([out.v_im[t] for t in range(4)]); keep.append(k)
        rc = lib().oracle_svd2_complex(n, a_re, a_im, u_re, u_im, v_re, v_im,
                                       _ptr(out.smax), _ptr(out.smin),
                                       _ptr(out.shift), mode, int(sine_form),
                                       threads, st)
    if rc != 0:
        raise ValueError("oracle rejected arguments (rc=%d)" % rc)
    return out


def backscale(smax, smin, shift, mode="safe"):
    smax, smin, shift = (np.ascontiguousarray(x, dtype=np.float64)
                         for x in (smax, smin, shift))
    n = smax.shape[0]
    o = [np.zeros(n) for _ in range(3)]
    lib().oracle_backscale(n, _ptr(smax), _ptr(smin), _ptr(shift),
                           MODES[mode], *[_ptr(x) for x in o])
    return tuple(o)


def getexp(x):
    return lib().oracle_getexp(float(x))


def scalef(x, e):
    return lib().oracle_scalef(float(x), float(e))


def hypot(a, b):
    return lib().oracle_hypot(float(a), float(b))


def invsqrt(a):
    return lib().oracle_invsqrt(float(a))


def hypot_vec(a, b):
    """lanes.hypot_lane elementwise (lanes.py:213-227)."""
    a, b = (np.ascontiguousarray(x, dtype=np.float64) for x in (a, b))
    out = np.empty_like(a)
    lib().oracle_hypot_vec(a.size, _ptr(a), _ptr(b), _ptr(out))
    return out


def phase_vec(re, im):
    """lanes.polar's (cos, sin) elementwise (lanes.py:248-270)."""
    re, im = (np.ascontiguousarray(x, dtype=np.float64) for x in (re, im))
    c, s = np.empty_like(re), np.empty_like(re)
    lib().oracle_phase_vec(re.size, _ptr(re), _ptr(im), _ptr(c), _ptr(s))
    return c, s
