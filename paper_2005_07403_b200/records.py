"""AoSoA-8 record files (the reference's on-disk test-file format).

Format (cli.py:1-25, 102-134): raw little-endian
binary64, eight matrices per record.  A real record is 4 consecutive 8-lane
vectors e11, e21, e12, e22 (256 B); a complex record is 8 vectors with re/im
interleaved per entry, e11re, e11im, e21re, ... (512 B).  Matrix k lives in
lane k % 8 of record k // 8.

``read_testfile`` mirrors ``lanesvd.cli.read_testfile`` (SoA trains on the
host).  ``read_records`` keeps the record layout, and ``run_records``
decomposes records on the GPU without a repack pass: the streaming kernels
fetch 32-record blocks through their TMA ring and pick each lane's
components out of the record layout in shared memory
(``b2s_svd2_{real,complex}_records``).
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .layout import LANE_WIDTH, SvdBatchOut, is_device_array, padded_len

__all__ = ["DataError", "VECS_PER_RECORD", "read_testfile", "read_records",
           "records_to_trains", "trains_to_records", "write_testfile",
           "run_records"]

VECS_PER_RECORD = {"real": 4, "complex": 8}


class DataError(Exception):
    """Malformed or inconsistent input data (cli.py:56-57)."""


def _field(field):
    if field not in VECS_PER_RECORD:
        raise DataError("unknown field %r" % (field,))
    return VECS_PER_RECORD[field]


def read_records(path, field):
    """Validated (n_records, vecs, 8) float64 array of a test file.

    Raises DataError -- as lanesvd.cli.read_testfile does (cli.py:102-134)
    -- when the file cannot be opened, holds no data, is not a whole number
    of records, or contains a NaN or an infinity."""
    vecs = _field(field)
    rec_doubles = vecs * LANE_WIDTH
    try:
        size = os.stat(path).st_size
        data = np.fromfile(path, dtype="<f8") if size else np.empty(0)
    except OSError as exc:
        raise DataError("cannot read %s: %s" % (path, exc))
    if size == 0:
        raise DataError("%s is empty" % path)
    n_rec, extra = divmod(size, rec_doubles * 8)
    if extra:
        raise DataError("%s: %d bytes is not a multiple of the %d-byte %s record"
                        % (path, size, rec_doubles * 8, field))
    finite = np.isfinite(data)
    if not finite.all():
        raise DataError("%s: non-finite value at element %d"
                        % (path, int(np.argmin(finite))))
    return data.astype(np.float64, copy=False).reshape(n_rec, vecs, LANE_WIDTH)


def records_to_trains(recs, field):
    """(re, im) SoA trains of shape (4, n) from a record array."""
    vecs = _field(field)
    recs = np.asarray(recs).reshape(-1, vecs, LANE_WIDTH)
    if field == "real":
        return np.ascontiguousarray(recs.transpose(1, 0, 2).reshape(4, -1)), None
    re = np.ascontiguousarray(recs[:, 0::2, :].transpose(1, 0, 2).reshape(4, -1))
    im = np.ascontiguousarray(recs[:, 1::2, :].transpose(1, 0, 2).reshape(4, -1))
    return re, im


def trains_to_records(re, im=None):
    """Record array from (4, n) trains (n padded to a multiple of 8 with
    zeros)."""
    re = np.asarray(re, dtype=np.float64)
    n = re.shape[1]
    n_hat = padded_len(n)
    k = n_hat // LANE_WIDTH
    pad = lambda a: np.concatenate([a, np.zeros((4, n_hat - n))], axis=1)
    r = pad(re).reshape(4, k, LANE_WIDTH).transpose(1, 0, 2)
    if im is None:
        return np.ascontiguousarray(r)
    i = pad(np.asarray(im, dtype=np.float64)).reshape(4, k, LANE_WIDTH).transpose(1, 0, 2)
    out = np.empty((k, 8, LANE_WIDTH))
    out[:, 0::2] = r
    out[:, 1::2] = i
    return out


def read_testfile(path, field):
    """(re, im) trains of a test file, like lanesvd.cli.read_testfile."""
    return records_to_trains(read_records(path, field), field)


def write_testfile(path, re, im=None):
    """Write (4, n) trains as a record file (n padded to whole records)."""
    trains_to_records(re, im).astype("<f8", copy=False).tofile(path)


def run_records(records, n, field, backscale_mode="none", sine_form=False,
                device=None):
    """Decompose the first n matrices of a record array on the GPU.

    ``records``: (n_rec, vecs, 8) NumPy array (copied to the device) or a
    CUDA tensor already in HBM.  Returns an ``SvdBatchOut`` of SoA trains
    in HBM (``.cpu()`` for host arrays)."""
    import torch
    vecs = _field(field)
    if backscale_mode not in _lib.BACKSCALE:
        raise ValueError("unknown backscale mode %r" % (backscale_mode,))
    n = int(n)
    if n < 0:
        raise ValueError("negative batch size")
    if device is None:
        device = records.device if is_device_array(records) else \
            torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    rec = records.to(device=device, dtype=torch.float64) if is_device_array(records) \
        else torch.from_numpy(np.ascontiguousarray(records, dtype=np.float64)).to(device)
    rec = rec.reshape(-1).contiguous()
    if rec.numel() < -(-n // LANE_WIDTH) * vecs * LANE_WIDTH:
        raise ValueError("records hold fewer than n matrices")
    _lib.assert_device_fp_env(device.index or 0)
    cplx = field == "complex"
    out = SvdBatchOut.empty(n, cplx, device=device)
    rows = lambda a: _lib.ptr_array([a[t].data_ptr() for t in range(4)])
    u, _k1 = rows(out.u_re)
    v, _k2 = rows(out.v_re)
    stream = torch.cuda.current_stream(rec.device).cuda_stream
    flags = _lib.FLAG_SINE_FORM if sine_form else 0
    mode = _lib.BACKSCALE[backscale_mode]
    n_hat = out.n_hat          # whole records: padding lanes decompose as zero matrices
    with torch.cuda.device(device):
        _launch_records(cplx, n_hat, rec, out, u, v, rows, mode, flags, stream)
    return out


def _launch_records(cplx, n_hat, rec, out, u, v, rows, mode, flags, stream):
    if not cplx:
        rc = _lib.lib.b2s_svd2_real_records(n_hat, rec.data_ptr(), u, v,
                                            out.smax.data_ptr(), out.smin.data_ptr(),
                                            out.shift.data_ptr(), mode, flags, stream)
        _lib.check(rc, "b2s_svd2_real_records")
    else:
        ui, _k3 = rows(out.u_im)
        vi, _k4 = rows(out.v_im)
        rc = _lib.lib.b2s_svd2_complex_records(n_hat, rec.data_ptr(), u, ui, v, vi,
                                               out.smax.data_ptr(), out.smin.data_ptr(),
                                               out.shift.data_ptr(), mode, flags, stream)
        _lib.check(rc, "b2s_svd2_complex_records")
