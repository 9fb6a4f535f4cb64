"""Batch execution on B200 GPUs (drop-in for lanesvd.driver).

``run_batch`` keeps the reference contract (driver.py:149-190): it takes a
``Batch2x2`` and a ``RunConfig``, allocates the output, decomposes every
lane (padding lanes included) and returns ``(SvdBatchOut, wall_seconds)``
with the wall time covering only the decomposition.

Where the reference splits the padded lane range into contiguous
chunk-aligned slabs, one per CPU thread (driver.py:134-146), this engine
splits it into contiguous shards, one per GPU, each processed by one fused
kernel.  Host (NumPy) batches are streamed through each GPU with the
pipelined host-buffer C-ABI; device-resident batches are processed in HBM.
Every path runs the same kernel, so results are bit-identical across paths,
shard counts and partitions, as in the reference.
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import svd2 as _svd2
from .layout import (LANE_WIDTH, Batch2x2, SvdBatchOut, from_trains, pack,
                     unpack)

__all__ = ["RunConfig", "run_batch", "run_batch_into", "svd2_chunk",
           "svd2_single", "shards",
           "FIELDS", "PATHS", "BACKSCALE_MODES"]

FIELDS = ("real", "complex")
# "cuda" is the engine's path; the reference's CPU path names are accepted
# for drop-in compatibility and run the same kernel (results are defined to be
# bit-identical across paths, driver.py:1-10).
PATHS = ("cuda", "vectorized", "pointwise")
BACKSCALE_MODES = ("none", "safe", "unconditional")

# Shard boundaries are multiples of this many lanes (2 KiB per train), so
# every shard starts vector- and sector-aligned.
SHARD_ALIGN = 256


@dataclass(frozen=True)
class RunConfig:
    """How a batch run executes (driver.py:37-63).

    ``devices``: CUDA device ordinals to shard over (None = the current
    device).  ``threads`` is kept for signature compatibility: 0 means one
    host worker per shard.  ``chunk``: lanes per host-pipeline chunk (0 =
    library default)."""
    field: str = "real"
    path: str = "cuda"
    threads: int = 0
    backscale_mode: str = "none"
    devices: tuple | None = None
    chunk: int = 0

    def __post_init__(self):
        if self.field not in FIELDS:
            raise ValueError("field must be one of %r" % (FIELDS,))
        if self.path not in PATHS:
            raise ValueError("path must be one of %r" % (PATHS,))
        if self.backscale_mode not in BACKSCALE_MODES:
            raise ValueError("backscale_mode must be one of %r"
                             % (BACKSCALE_MODES,))
        if self.threads < 0:
            raise ValueError("threads must be >= 0")
        if self.chunk < 0:
            raise ValueError("chunk must be >= 0")
        if self.devices is not None:
            if len(self.devices) == 0:
                raise ValueError("devices must be non-empty")
            if any(int(d) < 0 for d in self.devices):
                raise ValueError("device ordinals must be >= 0")

    @property
    def device_list(self):
        if self.devices is not None:
            return tuple(int(d) for d in self.devices)
        import torch
        return (torch.cuda.current_device(),)

    @property
    def worker_count(self):
        return len(self.device_list)


def shards(n_hat, parts, align=SHARD_ALIGN):
    """Contiguous ``align``-lane-aligned spans covering [0, n_hat), near
    equal, one per part (the GPU analogue of driver._slabs, 134-146).
    Empty spans are dropped; the last span absorbs the ragged tail."""
    n_hat = int(n_hat)
    if n_hat == 0:
        return []
    units = -(-n_hat // align)
    parts = max(1, min(int(parts), units))
    base, extra = divmod(units, parts)
    spans, lo = [], 0
    for w in range(parts):
        hi = min(n_hat, lo + (base + (1 if w < extra else 0)) * align)
        if hi > lo:
            spans.append((lo, hi))
        lo = hi
    return spans


def _host_shard(batch, out, lo, hi, mode, flags, device, chunk):
    """One GPU streams host lanes [lo, hi) through the host-buffer C-ABI."""
    n = hi - lo
    addr = lambda a: a.ctypes.data + lo * 8
    a, _k1 = _lib.ptr_array([addr(batch.re[t]) for t in range(4)])
    u, _k2 = _lib.ptr_array([addr(out.u_re[t]) for t in range(4)])
    v, _k3 = _lib.ptr_array([addr(out.v_re[t]) for t in range(4)])
    sm, sn, sh = addr(out.smax), addr(out.smin), addr(out.shift)
    if batch.im is None:
        rc = _lib.lib.b2s_svd2_real_host(n, a, u, v, sm, sn, sh, mode, flags,
                                         device, chunk)
        _lib.check(rc, "b2s_svd2_real_host")
        return
    ai, _k4 = _lib.ptr_array([addr(batch.im[t]) for t in range(4)])
    ui, _k5 = _lib.ptr_array([addr(out.u_im[t]) for t in range(4)])
    vi, _k6 = _lib.ptr_array([addr(out.v_im[t]) for t in range(4)])
    rc = _lib.lib.b2s_svd2_complex_host(n, a, ai, u, ui, v, vi, sm, sn, sh,
                                        mode, flags, device, chunk)
    _lib.check(rc, "b2s_svd2_complex_host")


def _device_out_dict(out, lo, hi):
    sl = lambda t: None if t is None else [t[k][lo:hi] for k in range(4)]
    return {"u_re": sl(out.u_re), "u_im": sl(out.u_im),
            "v_re": sl(out.v_re), "v_im": sl(out.v_im),
            "smax": out.smax[lo:hi], "smin": out.smin[lo:hi],
            "shift": out.shift[lo:hi]}


def _host_trains_ok(batch):
    for a in ((batch.re,) if batch.im is None else (batch.re, batch.im)):
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64
                and a.flags.c_contiguous):
            return False
    return True


def _check_host_out(out, n_hat):
    """Caller-owned host outputs: float64, C-contiguous, the batch's shape
    (the C-ABI writes through raw pointers)."""
    for name, arr in out.trains().items():
        want = (n_hat,) if name in ("smax", "smin", "shift") else (4, n_hat)
        if not isinstance(arr, np.ndarray) or arr.dtype != np.float64:
            raise ValueError("output %s must be a float64 NumPy array" % name)
        if tuple(arr.shape) != want:
            raise ValueError("output %s must have shape %r, got %r"
                             % (name, want, tuple(arr.shape)))
        if not arr.flags.c_contiguous or not arr.flags.writeable:
            raise ValueError("output %s must be C-contiguous and writeable" % name)


def run_batch(batch, cfg, sine_form=False, dump_states_to=None):
    """Decompose a whole batch (driver.py:149-190) on the GPU(s).

    Returns ``(SvdBatchOut, wall_time_seconds)``; outputs live where the
    inputs live (host NumPy or HBM).  ``dump_states_to`` writes the
    intermediate phase trains as raw little-endian float64 in the order of
    driver._dump_states (driver.py:193-216), outside the timed region."""
    if not isinstance(batch, Batch2x2):
        raise TypeError("expected a Batch2x2")
    if batch.field != cfg.field:
        raise ValueError("batch field %r does not match config field %r"
                         % (batch.field, cfg.field))
    out = SvdBatchOut.empty(batch.n, batch.im is not None,
                            device=batch.re.device if batch.on_device else None)
    wall = run_batch_into(batch, out, cfg, sine_form=sine_form)
    if dump_states_to is not None:
        _dump_states(dump_states_to, batch, sine_form)
    return out, wall


def run_batch_into(batch, out, cfg, sine_form=False):
    """``run_batch`` into caller-owned output trains (e.g. pinned host
    memory, or preallocated HBM), returning the wall time in seconds.

    Host batches stream through every device of ``cfg`` (one contiguous
    shard per GPU, one host thread per GPU); device batches run in HBM on
    their own device, asynchronously ordered on torch's current stream and
    synchronised before returning."""
    if not isinstance(batch, Batch2x2):
        raise TypeError("expected a Batch2x2")
    if batch.field != cfg.field:
        raise ValueError("batch field %r does not match config field %r"
                         % (batch.field, cfg.field))
    cplx = batch.im is not None
    if (out.u_im is not None) != cplx or out.n_hat != batch.n_hat:
        raise ValueError("output trains do not match the batch")
    if out.on_device != batch.on_device:
        raise ValueError("outputs must live where the inputs live")
    mode = _lib.BACKSCALE[cfg.backscale_mode]
    flags = _lib.FLAG_SINE_FORM if sine_form else 0
    n_hat = batch.n_hat
    if batch.on_device:
        import torch
        device = batch.re.device
        _lib.assert_device_fp_env(device.index)
        in_re = [batch.re[t] for t in range(4)]
        in_im = [batch.im[t] for t in range(4)] if cplx else None
        with torch.cuda.device(device):
            torch.cuda.synchronize(device)
            t0 = time.perf_counter()
            _svd2.launch_device(n_hat, in_re, in_im,
                                _device_out_dict(out, 0, n_hat), mode, flags)
            torch.cuda.synchronize(device)
            return time.perf_counter() - t0
    _check_host_out(out, n_hat)
    if not _host_trains_ok(batch):
        batch = Batch2x2(n=batch.n, re=np.ascontiguousarray(batch.re, dtype=np.float64),
                         im=None if batch.im is None else
                         np.ascontiguousarray(batch.im, dtype=np.float64))
    devices = cfg.device_list
    for d in devices:
        _lib.assert_device_fp_env(d)
    spans = shards(n_hat, len(devices))
    work = [(lo, hi, devices[k]) for k, (lo, hi) in enumerate(spans)]
    run = lambda w: _host_shard(batch, out, w[0], w[1], mode, flags,
                                w[2], cfg.chunk)
    t0 = time.perf_counter()
    if len(work) <= 1:
        for w in work:
            run(w)
    else:
        with ThreadPoolExecutor(max_workers=len(work)) as pool:
            list(pool.map(run, work))
    return time.perf_counter() - t0


def _dump_states(path, batch, sine_form):
    """Raw binary64 state trains, driver.py:193-216 order (outside timing)."""
    _, scale, urv, tri = _svd2.svd2_lanes(batch.parts(), sine_form=sine_form,
                                          with_states=True)
    with open(path, "wb") as fh:
        for train in _svd2.dump_trains(scale, urv, tri):
            arr = train.cpu().numpy() if hasattr(train, "cpu") else train
            np.ascontiguousarray(arr, dtype="<f8").tofile(fh)


def svd2_chunk(re_chunk, im_chunk=None, sine_form=False):
    """Decompose one aligned chunk of exactly 8 matrices (driver.py:88-106);
    returns an ``SvdBatchOut`` of 8 lanes, not backscaled."""
    re_chunk = np.asarray(re_chunk, dtype=np.float64)
    if re_chunk.shape != (4, LANE_WIDTH):
        raise ValueError("chunk must be (4, %d), got %r"
                         % (LANE_WIDTH, (re_chunk.shape,)))
    if im_chunk is not None:
        im_chunk = np.asarray(im_chunk, dtype=np.float64)
        if im_chunk.shape != (4, LANE_WIDTH):
            raise ValueError("re/im chunk shapes differ")
    batch = from_trains(re_chunk, im_chunk)
    cfg = RunConfig(field=batch.field)
    out, _ = run_batch(batch, cfg, sine_form=sine_form)
    return out


def svd2_single(a, sine_form=False):
    """Decompose one 2x2 matrix (driver.py:109-131); returns a
    ``MatrixSvd`` with scaled singular values and the shift."""
    a = np.asarray(a)
    if a.shape != (2, 2):
        raise ValueError("expected a 2x2 matrix, got shape %r" % (a.shape,))
    batch = pack(a.reshape(1, 2, 2))
    out, _ = run_batch(batch, RunConfig(field=batch.field),
                       sine_form=sine_form)
    return unpack(out)[0]
