"""Structure-of-arrays batch containers (drop-in for lanesvd.layout).

Same layout contract as the reference (layout.py:1-16): a batch of n
matrices is a C-contiguous (4, n_hat) float64 array whose rows are the
entry trains e11, e21, e12, e22 (column-major entry order); complex batches
carry a second (4, n_hat) array of imaginary parts.  n_hat = ceil(n/8)*8 and
padding lanes hold zeros, which decompose as zero matrices (sigma 0,
shift DBL_MAX, U = V = I).

B200 additions: trains may live in HBM as CUDA ``torch.Tensor`` objects
(``Batch2x2.to(device)``); host trains are 64-byte aligned NumPy arrays
exactly as in the reference, and the host path streams them through the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

__all__ = [
    "LANE_WIDTH", "padded_len", "aligned_zeros", "Batch2x2", "SvdBatchOut",
    "MatrixSvd", "pack", "unpack", "from_trains", "unpack_inputs",
    "is_device_array",
]

LANE_WIDTH = 8            # lanes.py:38; n_hat granularity
_ALIGN = 64
_ENTRY_ORDER = ((0, 0), (1, 0), (0, 1), (1, 1))   # e11, e21, e12, e22


def padded_len(n):
    """Smallest multiple of LANE_WIDTH >= n (layout.py:33-37)."""
    n = int(n)
    if n < 0:
        raise ValueError("negative batch size")
    return (n + LANE_WIDTH - 1) // LANE_WIDTH * LANE_WIDTH


def aligned_zeros(rows, cols):
    """Zeroed C-contiguous (rows, cols) float64 host array whose rows all
    start on a 64-byte boundary (layout.py:40-51)."""
    if cols % LANE_WIDTH:
        raise ValueError("column count must be a multiple of %d" % LANE_WIDTH)
    count = rows * cols
    raw = np.zeros(count + _ALIGN // 8, dtype=np.float64)
    skip = ((-raw.ctypes.data) % _ALIGN) // 8
    return raw[skip:skip + count].reshape(rows, cols)


def is_device_array(x):
    """True for a CUDA torch tensor (trains resident in HBM)."""
    return getattr(x, "is_cuda", False) is True


def _device_zeros(shape, device):
    import torch
    return torch.zeros(shape, dtype=torch.float64, device=device)


def _device_empty(shape, device):
    import torch
    return torch.empty(shape, dtype=torch.float64, device=device)


class MatrixSvd(NamedTuple):
    """One unpacked result (layout.py:54-66): u, v (2, 2) arrays and the
    stored smax, smin, shift lane values."""
    u: np.ndarray
    v: np.ndarray
    smax: float
    smin: float
    shift: float


@dataclass
class Batch2x2:
    """Input batch: n genuine lanes inside (4, n_hat) trains (layout.py:69-103).

    ``re``/``im`` are host NumPy arrays or CUDA tensors (both the same kind).
    """
    n: int
    re: object
    im: object = None

    def __post_init__(self):
        shape = tuple(self.re.shape)
        if len(shape) != 2 or shape[0] != 4 or shape[1] % LANE_WIDTH:
            raise ValueError("trains must be (4, multiple of %d), got %r"
                             % (LANE_WIDTH, shape))
        if self.im is not None:
            if tuple(self.im.shape) != shape:
                raise ValueError("re/im train shapes differ")
            if is_device_array(self.im) != is_device_array(self.re):
                raise ValueError("re/im trains must both be host or device")
        if not 0 <= self.n <= shape[1]:
            raise ValueError("n outside the padded train length")

    @property
    def n_hat(self):
        return int(self.re.shape[1])

    @property
    def field(self):
        return "real" if self.im is None else "complex"

    @property
    def on_device(self):
        return is_device_array(self.re)

    def parts(self):
        """Component trains in kernel order (re/im interleaved per entry)."""
        if self.im is None:
            return tuple(self.re[t] for t in range(4))
        return tuple(x for t in range(4) for x in (self.re[t], self.im[t]))

    def to(self, device):
        """Copy the trains into HBM on ``device`` (bit-exact)."""
        import torch

        def mv(a):
            if not is_device_array(a):
                a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            return a.to(device=device, dtype=torch.float64).contiguous()
        return Batch2x2(n=self.n, re=mv(self.re),
                        im=None if self.im is None else mv(self.im))

    def cpu(self):
        if not self.on_device:
            return self
        re = aligned_zeros(4, self.n_hat)
        re[:] = self.re.cpu().numpy()
        im = None
        if self.im is not None:
            im = aligned_zeros(4, self.n_hat)
            im[:] = self.im.cpu().numpy()
        return Batch2x2(n=self.n, re=re, im=im)


@dataclass
class SvdBatchOut:
    """Output batch, same layout as the input (layout.py:106-130)."""
    n: int
    u_re: object
    u_im: object
    v_re: object
    v_im: object
    smax: object
    smin: object
    shift: object

    @property
    def n_hat(self):
        return int(self.u_re.shape[1])

    @property
    def on_device(self):
        return is_device_array(self.u_re)

    @classmethod
    def empty(cls, n, complex_field, device=None):
        """Allocate output trains: aligned host arrays, or HBM tensors when
        ``device`` names a CUDA device (uninitialised; every lane is written)."""
        n_hat = padded_len(n)
        if device is None:
            mk = lambda: aligned_zeros(4, n_hat)
            vec = lambda: aligned_zeros(1, n_hat)[0]
        else:
            mk = lambda: _device_empty((4, n_hat), device)
            vec = lambda: _device_empty((n_hat,), device)
        return cls(n=n, u_re=mk(), u_im=mk() if complex_field else None,
                   v_re=mk(), v_im=mk() if complex_field else None,
                   smax=vec(), smin=vec(), shift=vec())

    def trains(self):
        """Named output trains (u/v blocks are (4, n_hat))."""
        out = {"u_re": self.u_re, "v_re": self.v_re, "smax": self.smax,
               "smin": self.smin, "shift": self.shift}
        if self.u_im is not None:
            out["u_im"] = self.u_im
            out["v_im"] = self.v_im
        return out

    def cpu(self):
        """Host copy (NumPy) of a device-resident result."""
        if not self.on_device:
            return self
        cv = lambda a: None if a is None else a.cpu().numpy()
        return SvdBatchOut(n=self.n, u_re=cv(self.u_re), u_im=cv(self.u_im),
                           v_re=cv(self.v_re), v_im=cv(self.v_im),
                           smax=cv(self.smax), smin=cv(self.smin),
                           shift=cv(self.shift))


def _reject_nonfinite(a, what):
    if not np.isfinite(a).all():
        raise ValueError("non-finite value in %s" % what)


def pack(matrices):
    """(n, 2, 2) real or complex matrices -> aligned padded Batch2x2, values
    copied bit-exactly; non-finite entries rejected (layout.py:138-165)."""
    a = np.asarray(matrices)
    if a.ndim != 3 or a.shape[1:] != (2, 2):
        raise ValueError("expected shape (n, 2, 2), got %r" % (a.shape,))
    n = a.shape[0]
    n_hat = padded_len(n)
    cplx = np.iscomplexobj(a)
    if cplx:
        a = a.astype(np.complex128, copy=False)
        _reject_nonfinite(a.real, "matrix real parts")
        _reject_nonfinite(a.imag, "matrix imaginary parts")
    else:
        a = a.astype(np.float64, copy=False)
        _reject_nonfinite(a, "matrix entries")
    re = aligned_zeros(4, n_hat)
    im = aligned_zeros(4, n_hat) if cplx else None
    for t, (i, j) in enumerate(_ENTRY_ORDER):
        if cplx:
            re[t, :n] = a[:, i, j].real
            im[t, :n] = a[:, i, j].imag
        else:
            re[t, :n] = a[:, i, j]
    return Batch2x2(n=n, re=re, im=im)


def from_trains(re, im=None, n=None):
    """Batch from train-ordered (4, m) arrays, copied into aligned padded
    trains; non-finite genuine lanes rejected (layout.py:168-189)."""
    re = np.asarray(re, dtype=np.float64)
    if re.ndim != 2 or re.shape[0] != 4:
        raise ValueError("expected (4, n) trains, got %r" % (re.shape,))
    m = re.shape[1] if n is None else int(n)
    _reject_nonfinite(re[:, :m], "matrix entries")
    out_re = aligned_zeros(4, padded_len(m))
    out_re[:, :m] = re[:, :m]
    out_im = None
    if im is not None:
        im = np.asarray(im, dtype=np.float64)
        if im.shape != re.shape:
            raise ValueError("re/im train shapes differ")
        _reject_nonfinite(im[:, :m], "matrix imaginary parts")
        out_im = aligned_zeros(4, padded_len(m))
        out_im[:, :m] = im[:, :m]
    return Batch2x2(n=m, re=out_re, im=out_im)


def _matrices(re, im, n):
    """(n, 2, 2) matrices from (4, >=n) trains."""
    if im is None:
        m = np.empty((n, 2, 2), dtype=np.float64)
    else:
        m = np.empty((n, 2, 2), dtype=np.complex128)
    for t, (i, j) in enumerate(_ENTRY_ORDER):
        if im is None:
            m[:, i, j] = re[t, :n]
        else:
            m[:, i, j].real = re[t, :n]
            m[:, i, j].imag = im[t, :n]
    return m


def unpack(out):
    """Per-matrix records of the n genuine lanes (layout.py:206-224)."""
    out = out.cpu()
    u = _matrices(out.u_re, out.u_im, out.n)
    v = _matrices(out.v_re, out.v_im, out.n)
    return [MatrixSvd(u=u[k], v=v[k], smax=float(out.smax[k]),
                      smin=float(out.smin[k]), shift=float(out.shift[k]))
            for k in range(out.n)]


def unpack_inputs(batch):
    """(n, 2, 2) array of the genuine input matrices (layout.py:227-238)."""
    batch = batch.cpu()
    return _matrices(batch.re, batch.im, batch.n)
