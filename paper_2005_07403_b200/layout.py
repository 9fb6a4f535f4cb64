"""Batch containers for the SoA trains (drop-in for lanesvd.layout).

The contract is the reference's (layout.py:1-16): n matrices live in a
C-contiguous (4, n_hat) float64 block whose rows are the entry trains in
column-major entry order -- e11, e21, e12, e22 -- with lane k of every row
belonging to matrix k; a complex batch carries a second block of imaginary
parts.  n_hat = ceil(n / 8) * 8, and padding lanes are zeros (they come out
as zero-matrix results: sigma 0, shift DBL_MAX, U = V = I).

On B200 the blocks may also be CUDA tensors resident in HBM
(``Batch2x2.to(device)``, ``SvdBatchOut.empty(..., device=...)``); host
blocks are 64-byte aligned NumPy arrays, as the reference allocates them.
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

LANE_WIDTH = 8                  # lanes.py:38: batches are whole 8-lane chunks
ROW_ALIGN_BYTES = 64
# train t holds matrix entry ENTRIES[t] = (row, col)
ENTRIES = ((0, 0), (1, 0), (0, 1), (1, 1))


def padded_len(n):
    """n rounded up to a whole number of LANE_WIDTH-lane chunks
    (layout.py:33-37); ValueError for n < 0."""
    n = int(n)
    if n < 0:
        raise ValueError("negative batch size")
    chunks, rest = divmod(n, LANE_WIDTH)
    return (chunks + (rest > 0)) * LANE_WIDTH


def aligned_zeros(rows, cols):
    """(rows, cols) float64 zeros, C order, every row on a 64-byte boundary
    (layout.py:40-51): the block starts aligned and a row is a whole number
    of 8-double chunks."""
    if cols % LANE_WIDTH:
        raise ValueError("column count must be a multiple of %d" % LANE_WIDTH)
    slack = ROW_ALIGN_BYTES // 8
    store = np.zeros(rows * cols + slack, dtype=np.float64)
    lead = (-store.ctypes.data % ROW_ALIGN_BYTES) // 8
    return store[lead:lead + rows * cols].reshape(rows, cols)


def is_device_array(x):
    """True for a CUDA torch tensor (trains resident in HBM)."""
    return getattr(x, "is_cuda", False) is True


def _hbm_block(shape, device):
    import torch
    return torch.empty(shape, dtype=torch.float64, device=device)


def _to_host(x):
    return None if x is None else (x.cpu().numpy() if is_device_array(x) else x)


class MatrixSvd(NamedTuple):
    """One matrix's result (layout.py:54-66): U, V as (2, 2) arrays and the
    lane's stored smax, smin, shift."""
    u: np.ndarray
    v: np.ndarray
    smax: float
    smin: float
    shift: float


def _check_blocks(n, re, im):
    shape = tuple(re.shape)
    well_formed = len(shape) == 2 and shape[0] == 4 and shape[1] % LANE_WIDTH == 0
    if not well_formed:
        raise ValueError("trains must be (4, multiple of %d), got %r" % (LANE_WIDTH, shape))
    if im is not None and tuple(im.shape) != shape:
        raise ValueError("re/im train shapes differ")
    if im is not None and is_device_array(im) != is_device_array(re):
        raise ValueError("re/im trains must both be host or device")
    if n < 0 or n > shape[1]:
        raise ValueError("n outside the padded train length")


@dataclass
class Batch2x2:
    """An input batch: ``n`` genuine lanes in (4, n_hat) train blocks
    (layout.py:69-103).  ``re``/``im``: host arrays or CUDA tensors."""
    n: int
    re: object
    im: object = None

    def __post_init__(self):
        _check_blocks(self.n, self.re, self.im)

    @property
    def n_hat(self):
        return int(self.re.shape[1])

    @property
    def field(self):
        return "complex" if self.im is not None else "real"

    @property
    def on_device(self):
        return is_device_array(self.re)

    def parts(self):
        """The component trains in kernel order: e11, e21, e12, e22, or for
        complex batches e11re, e11im, e21re, ... (svd2.py:521-570)."""
        blocks = (self.re,) if self.im is None else (self.re, self.im)
        return tuple(b[t] for t in range(4) for b in blocks)

    def to(self, device):
        """A copy with both blocks in HBM on ``device`` (bit-exact)."""
        import torch

        def upload(block):
            t = block if is_device_array(block) else torch.from_numpy(
                np.ascontiguousarray(block, dtype=np.float64))
            return t.to(device=device, dtype=torch.float64).contiguous()
        return Batch2x2(self.n, upload(self.re), None if self.im is None else upload(self.im))

    def cpu(self):
        """A host copy in aligned blocks (self when already on the host)."""
        if not self.on_device:
            return self

        def download(block):
            host = aligned_zeros(4, self.n_hat)
            np.copyto(host, block.cpu().numpy())
            return host
        return Batch2x2(self.n, download(self.re), None if self.im is None else download(self.im))


_OUT_NAMES = ("u_re", "u_im", "v_re", "v_im", "smax", "smin", "shift")


@dataclass
class SvdBatchOut:
    """Output trains in the input's layout (layout.py:106-130): U and V as
    (4, n_hat) blocks (imaginary blocks None for real batches), smax, smin
    and shift as (n_hat,) vectors."""
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
        """Output storage for n lanes: zeroed aligned host blocks, or
        uninitialised HBM tensors on ``device`` (every lane is written)."""
        n_hat = padded_len(n)
        if device is None:
            block = lambda: aligned_zeros(4, n_hat)
            vector = lambda: aligned_zeros(1, n_hat)[0]
        else:
            block = lambda: _hbm_block((4, n_hat), device)
            vector = lambda: _hbm_block((n_hat,), device)
        cplx = bool(complex_field)
        return cls(n, block(), block() if cplx else None, block(), block() if cplx else None,
                   vector(), vector(), vector())

    def trains(self):
        """Output trains by name; the imaginary blocks only when present."""
        return {k: getattr(self, k) for k in _OUT_NAMES if getattr(self, k) is not None}

    def cpu(self):
        """Host (NumPy) copy of a device-resident result."""
        if not self.on_device:
            return self
        return SvdBatchOut(self.n, *(_to_host(getattr(self, k)) for k in _OUT_NAMES))


def _require_finite(values, what):
    if not np.all(np.isfinite(values)):
        raise ValueError("non-finite value in %s" % what)


def pack(matrices):
    """(n, 2, 2) real or complex matrices into an aligned padded batch,
    values copied bit-exactly, non-finite entries rejected
    (layout.py:138-165)."""
    a = np.asarray(matrices)
    if a.ndim != 3 or a.shape[1:] != (2, 2):
        raise ValueError("expected shape (n, 2, 2), got %r" % (a.shape,))
    n = a.shape[0]
    if np.iscomplexobj(a):
        a = a.astype(np.complex128, copy=False)
        _require_finite(a.real, "matrix real parts")
        _require_finite(a.imag, "matrix imaginary parts")
        components = (a.real, a.imag)
    else:
        a = a.astype(np.float64, copy=False)
        _require_finite(a, "matrix entries")
        components = (a,)
    blocks = []
    for comp in components:
        block = aligned_zeros(4, padded_len(n))
        # (n, 2, 2) -> (4, n) in column-major entry order
        block[:, :n] = comp.transpose(2, 1, 0).reshape(4, n)
        blocks.append(block)
    return Batch2x2(n, blocks[0], blocks[1] if len(blocks) > 1 else None)


def from_trains(re, im=None, n=None):
    """A batch from train-ordered (4, m) arrays (the first n lanes, default
    all), copied into aligned padded blocks; non-finite lanes rejected
    (layout.py:168-189)."""
    src = [np.asarray(re, dtype=np.float64)]
    if src[0].ndim != 2 or src[0].shape[0] != 4:
        raise ValueError("expected (4, n) trains, got %r" % (src[0].shape,))
    if im is not None:
        src.append(np.asarray(im, dtype=np.float64))
        if src[1].shape != src[0].shape:
            raise ValueError("re/im train shapes differ")
    m = src[0].shape[1] if n is None else int(n)
    what = ("matrix entries", "matrix imaginary parts")
    blocks = []
    for k, s in enumerate(src):
        _require_finite(s[:, :m], what[k])
        block = aligned_zeros(4, padded_len(m))
        np.copyto(block[:, :m], s[:, :m])
        blocks.append(block)
    return Batch2x2(m, blocks[0], blocks[1] if len(blocks) > 1 else None)


def _as_matrices(re, im, n):
    """(n, 2, 2) matrices from the first n lanes of (4, >= n) blocks (parts
    assigned separately: re + 1j * im would not keep signed zeros)."""
    out = np.empty((n, 2, 2), dtype=np.float64 if im is None else np.complex128)
    # out[k, i, j] <- train 2 j + i (column-major entry order)
    for t, (i, j) in enumerate(ENTRIES):
        if im is None:
            out[:, i, j] = re[t, :n]
        else:
            out[:, i, j].real = re[t, :n]
            out[:, i, j].imag = im[t, :n]
    return out


def unpack(out):
    """Per-matrix results of the n genuine lanes (layout.py:206-224)."""
    out = out.cpu()
    u = _as_matrices(out.u_re, out.u_im, out.n)
    v = _as_matrices(out.v_re, out.v_im, out.n)
    smax, smin, shift = (np.asarray(x)[:out.n].tolist() for x in (out.smax, out.smin, out.shift))
    return [MatrixSvd(u[k], v[k], smax[k], smin[k], shift[k]) for k in range(out.n)]


def unpack_inputs(batch):
    """The genuine input matrices as an (n, 2, 2) array (layout.py:227-238)."""
    batch = batch.cpu()
    return _as_matrices(batch.re, batch.im, batch.n)
