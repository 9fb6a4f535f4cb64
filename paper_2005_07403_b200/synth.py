"""Seeded, counter-based synthetic batches for the BASELINE configs.

Every value is a pure function of (seed, config, stream, lane), so any
contiguous lane range -- one GPU's shard, a parity window, the CPU baseline's
sample -- regenerates bit-identically here (NumPy) and on the device
(``csrc/b2s_synth.cu``, C-ABI ``b2s_synth``).  The reference has no public
benchmark suite; these distributions are BASELINE.json's config strings
restated:

0  real,    n = 65536, entries +-U[1,2) * 2^e, e uniform in [-20, 20]
1  complex, n = 2^20,  re/im independent, e in [-20, 20]
2  real,    n = 2^24,  e in [-1074, 1023] (subnormals included); ~10% each
   zero column / rank-1 / diagonal / upper-triangular, 60% dense
3  real,    n = 2^30,  e in [-100, 100]
4  complex, n = 2^28,  60% dense (config 1), 20% phase-rotated triangular,
   10% rank-deficient, 10% wide exponents [-1000, 1000]

Entry construction: x = (-1)^b * (1 + k 2^-52) * 2^e with 52 random mantissa
bits k, rounded once (ties to even) into the subnormal range when e < -1022.
Bits come from a SplitMix64 finaliser over a Weyl sequence keyed per
(seed, config, stream); exponents use the 64x64->high multiply map
(bias <= range / 2^64).
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    0: dict(field="real", n=1 << 16, lo=-20, hi=20),
    1: dict(field="complex", n=1 << 20, lo=-20, hi=20),
    2: dict(field="real", n=1 << 24, lo=-1074, hi=1023),
    3: dict(field="real", n=1 << 30, lo=-100, hi=100),
    4: dict(field="complex", n=1 << 28, lo=-20, hi=20),
}

_U = np.uint64
_M1 = _U(0xBF58476D1CE4E5B9)
_M2 = _U(0x94D049BB133111EB)
_GOLD = _U(0x9E3779B97F4A7C15)
_KC = _U(0xC2B2AE3D27D4EB4F)
_KS = _U(0x165667B19E3779F9)
_MANT = _U((1 << 52) - 1)

# stream ids (shared with b2s_synth.cu)
S_CLASS = 64
S_R1_SM, S_R1_E = 70, 71          # config 2 rank-1 multiplier
S_PH = 80                         # config 4 phases: 80..83
S_C4_C = 90                       # config 4 complex multiplier: 90..93
S_WIDE = 100                      # config 4 wide exponents: 100..107


def _mix(x):
    x = x ^ (x >> _U(30))
    x = x * _M1
    x = x ^ (x >> _U(27))
    x = x * _M2
    return x ^ (x >> _U(31))


def _key(seed, config, stream):
    with np.errstate(over="ignore"):
        k = (_U(seed) * _GOLD + _U(config) * _KC + _U(stream) * _KS + _U(1))
        return _mix(np.array([k], dtype=np.uint64))[0]


def draw(seed, config, stream, lanes):
    """64 random bits per lane (lanes: uint64 array of global lane ids)."""
    k = _key(seed, config, stream)
    return _mix(k + lanes * _GOLD)


def _mulhi_range(r, rng):
    """floor(r * rng / 2^64) for rng < 2^32 (exact, via 32-bit halves)."""
    rng = np.asarray(rng, dtype=np.uint64)
    h = r >> _U(32)
    lo = r & _U(0xFFFFFFFF)
    return (h * rng + ((lo * rng) >> _U(32))) >> _U(32)


def make_value(sm, e):
    """(-1)^b (1 + k 2^-52) 2^e from sign/mantissa bits ``sm`` and int64
    exponents ``e`` in [-1074, 1023]; one round-to-nearest-even into the
    subnormal range."""
    sign = (sm >> _U(63)) << _U(63)
    k = sm & _MANT
    e = np.asarray(e, dtype=np.int64)
    normal = e >= -1022
    out = np.empty(sm.shape, dtype=np.uint64)
    eb = (np.where(normal, e, 0) + 1023).astype(np.uint64)
    out[:] = sign | (eb << _U(52)) | k
    if not normal.all():
        idx = ~normal
        M = k[idx] | _U(1 << 52)
        sh = (-1022 - e[idx]).astype(np.uint64)       # 1..52
        q = M >> sh
        rem = M & ((_U(1) << sh) - _U(1))
        half = _U(1) << (sh - _U(1))
        up = (rem > half) | ((rem == half) & ((q & _U(1)) == _U(1)))
        q = q + up.astype(np.uint64)
        out[idx] = sign[idx] | q
    return out.view(np.float64)


def _val(seed, config, j, lanes, lo, hi, estream=None):
    sm = draw(seed, config, 2 * j, lanes)
    er = draw(seed, config, 2 * j + 1 if estream is None else estream, lanes)
    e = np.int64(lo) + _mulhi_range(er, hi - lo + 1).astype(np.int64)
    return make_value(sm, e)


def _cmul(ar, ai, br, bi):
    # plain complex product, no fma: (ar br - ai bi, ar bi + ai br)
    return ar * br - ai * bi, ar * bi + ai * br


def _phase(seed, config, stream, lanes):
    # rational unit phase ((1-t^2)/(1+t^2), 2t/(1+t^2)), t = j / 2^19 in [-1, 1)
    r = draw(seed, config, stream, lanes)
    t = ((r >> _U(44)).astype(np.int64) - (1 << 19)).astype(np.float64) * 2.0 ** -19
    tt = t * t
    den = 1.0 + tt
    return (1.0 - tt) / den, (t + t) / den


def generate(config, seed, lane0, n):
    """Lanes [lane0, lane0+n) of ``config``: returns (re, im) with re a
    (4, n) float64 array (e11, e21, e12, e22) and im (4, n) or None."""
    c = CONFIGS[config]
    lanes = np.arange(lane0, lane0 + n, dtype=np.uint64)
    lo, hi = c["lo"], c["hi"]
    with np.errstate(over="ignore", under="ignore", invalid="ignore"):
        if c["field"] == "real":
            re = np.stack([_val(seed, config, t, lanes, lo, hi) for t in range(4)])
            if config == 2:
                _structure_real(re, seed, lanes)
            return re, None
        comps = [_val(seed, config, j, lanes, lo, hi) for j in range(8)]
        re = np.stack(comps[0::2])
        im = np.stack(comps[1::2])
        if config == 4:
            _structure_complex(re, im, seed, lanes)
        return re, im


def lane_class(seed, config, lanes):
    r = draw(seed, config, S_CLASS, lanes)
    return _mulhi_range(r, 10).astype(np.int64), (r & _U(1)).astype(bool)


def _structure_real(re, seed, lanes):
    """config 2: classes 0 zero column, 1 rank-1, 2 diagonal, 3 upper."""
    cls, bit = lane_class(seed, 2, lanes)
    z = cls == 0
    zc1 = z & ~bit
    zc2 = z & bit
    re[0, zc1] = 0.0
    re[1, zc1] = 0.0
    re[2, zc2] = 0.0
    re[3, zc2] = 0.0
    r1 = cls == 1
    if r1.any():
        l1 = lanes[r1]
        # drawn exponents of column 1 (streams 1, 3), as in _val
        e11 = -1074 + _mulhi_range(draw(seed, 2, 1, l1), 2098).astype(np.int64)
        e21 = -1074 + _mulhi_range(draw(seed, 2, 3, l1), 2098).astype(np.int64)
        hi_e = np.minimum(1021 - np.maximum(e11, e21), 1023)
        er = draw(seed, 2, S_R1_E, l1)
        ep = -1074 + _mulhi_range(er, (hi_e + 1075).astype(np.uint64)).astype(np.int64)
        cmult = make_value(draw(seed, 2, S_R1_SM, l1), ep)
        re[2, r1] = cmult * re[0, r1]
        re[3, r1] = cmult * re[1, r1]
    dg = cls == 2
    re[1, dg] = 0.0
    re[2, dg] = 0.0
    up = cls == 3
    re[1, up] = 0.0


def _structure_complex(re, im, seed, lanes):
    """config 4: classes 0-5 dense, 6-7 phase-rotated triangular,
    8 rank-deficient, 9 wide exponents."""
    cls, _ = lane_class(seed, 4, lanes)
    tri = (cls == 6) | (cls == 7)
    if tri.any():
        l = lanes[tri]
        p1 = _phase(seed, 4, S_PH + 0, l)
        p2 = _phase(seed, 4, S_PH + 1, l)
        q1 = _phase(seed, 4, S_PH + 2, l)
        q2 = _phase(seed, 4, S_PH + 3, l)
        t11 = (re[0, tri], im[0, tri])
        t12 = (re[2, tri], im[2, tri])
        t22 = (re[3, tri], im[3, tri])
        a11 = _cmul(*_cmul(*p1, *t11), *q1)
        a12 = _cmul(*_cmul(*p1, *t12), *q2)
        a22 = _cmul(*_cmul(*p2, *t22), *q2)
        re[0, tri], im[0, tri] = a11
        re[2, tri], im[2, tri] = a12
        re[3, tri], im[3, tri] = a22
        re[1, tri] = 0.0
        im[1, tri] = 0.0
    rd = cls == 8
    if rd.any():
        l = lanes[rd]
        cr = _val(seed, 4, 45, l, -20, 20, estream=S_C4_C + 1)   # streams 90, 91
        ci = _val(seed, 4, 46, l, -20, 20, estream=S_C4_C + 3)   # streams 92, 93
        a12 = _cmul(cr, ci, re[0, rd], im[0, rd])
        a22 = _cmul(cr, ci, re[1, rd], im[1, rd])
        re[2, rd], im[2, rd] = a12
        re[3, rd], im[3, rd] = a22
    wd = cls == 9
    if wd.any():
        l = lanes[wd]
        for j in range(8):
            v = _val(seed, 4, j, l, -1000, 1000, estream=S_WIDE + j)
            (re if j % 2 == 0 else im)[j // 2, wd] = v


def generate_device(config, seed, lane0, n, device=None, n_hat=None):
    """Lanes [lane0, lane0+n) of ``config`` generated directly in HBM by the
    ``b2s_synth`` kernel.  Returns (re, im) CUDA tensors of shape
    (4, n_hat) (im None for real configs); lanes past n are zero padding."""
    import torch
    from . import _lib
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    n_hat = n if n_hat is None else n_hat
    cplx = CONFIGS[config]["field"] == "complex"
    mk = lambda: (torch.zeros if n_hat > n else torch.empty)(
        (4, n_hat), dtype=torch.float64, device=device)
    re = mk()
    im = mk() if cplx else None
    rp, _k1 = _lib.ptr_array([re[t].data_ptr() for t in range(4)])
    ip, _k2 = (_lib.ptr_array([im[t].data_ptr() for t in range(4)])
               if cplx else (None, None))
    stream = torch.cuda.current_stream(re.device).cuda_stream
    rc = _lib.lib.b2s_synth(int(config), int(seed), int(lane0), int(n), rp,
                            ip, stream)
    _lib.check(rc, "b2s_synth")
    return re, im
