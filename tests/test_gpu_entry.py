"""GPU: the width-1 / width-8 entry points, caller-buffer validation,
device selection and the in-process multi-device host path.

Reference behaviour mirrored: test_driver.py:88-102 (svd2_single equals
the svd2_chunk lane bit for bit), driver.py:134-146 / 180-187 (sharded
run over workers gives the same trains as one worker).
"""

import numpy as np
import pytest

from helpers import assert_bits_equal

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2005_07403_b200 as b2s  # noqa: E402
from paper_2005_07403_b200 import synth  # noqa: E402
from paper_2005_07403_b200.svd2 import launch_device  # noqa: E402

DEV = torch.device("cuda", 0)


def _mats(field, n, seed):
    rng = np.random.default_rng(seed)
    e = rng.integers(-60, 60, size=(n, 2, 2))
    m = rng.uniform(1, 2, size=(n, 2, 2)) * np.where(rng.random((n, 2, 2)) < 0.5, -1, 1)
    x = np.ldexp(m, e)
    if field == "complex":
        y = np.ldexp(rng.uniform(1, 2, size=(n, 2, 2)), rng.integers(-60, 60, size=(n, 2, 2)))
        x = x + 1j * y
    return x


@pytest.mark.parametrize("field", ["real", "complex"])
def test_single_equals_chunk_equals_batch_bitwise(field):
    """svd2_single (width 1) == svd2_chunk (width 8) == run_batch lane,
    every U/V entry, sigma and shift, bit for bit -- and all equal the
    oracle (the reference's test_single_matches_chunk_lane, extended)."""
    mats = _mats(field, 8, 31)
    batch = b2s.pack(mats)
    chunk = b2s.svd2_chunk(batch.re, batch.im)
    whole, _ = b2s.run_batch(batch, b2s.RunConfig(field=field))
    ref = oracle.svd2(batch.re, batch.im)
    for name, arr in ref.trains().items():
        assert_bits_equal(chunk.trains()[name], arr, "chunk " + name)
        assert_bits_equal(whole.trains()[name], arr, "batch " + name)
    for k in range(8):
        one = b2s.svd2_single(mats[k])
        lane = b2s.unpack(chunk)[k]
        assert_bits_equal(np.array([one.smax, one.smin, one.shift]),
                          np.array([lane.smax, lane.smin, lane.shift]), "sigma lane %d" % k)
        assert_bits_equal(np.ascontiguousarray(one.u).view(np.float64), np.ascontiguousarray(lane.u).view(np.float64), "u lane %d" % k)
        assert_bits_equal(np.ascontiguousarray(one.v).view(np.float64), np.ascontiguousarray(lane.v).view(np.float64), "v lane %d" % k)


def _outd(out):
    return {"u_re": list(out.u_re), "u_im": None if out.u_im is None else list(out.u_im),
            "v_re": list(out.v_re), "v_im": None if out.v_im is None else list(out.v_im),
            "smax": out.smax, "smin": out.smin, "shift": out.shift}


@pytest.mark.parametrize("bad", ["f32_in", "strided_in", "short_out", "host_out", "f32_out",
                                 "missing_im", "state_count"])
def test_launch_device_rejects_bad_buffers(bad):
    """A float32, strided, short or host buffer raises ValueError before
    its pointer reaches the C-ABI (out-of-bounds HBM access)."""
    n = 4096
    re, _ = synth.generate_device(3, 1, 0, n, device=DEV)
    ins = [re[t] for t in range(4)]
    out = b2s.SvdBatchOut.empty(n, False, device=DEV)
    outd = _outd(out)
    states = None
    if bad == "f32_in":
        ins[2] = ins[2].float()
    elif bad == "strided_in":
        ins[1] = torch.zeros(2 * n, dtype=torch.float64, device=DEV)[::2]
    elif bad == "short_out":
        outd["smin"] = out.smin[: n // 2]
    elif bad == "host_out":
        outd["v_re"][3] = torch.zeros(n, dtype=torch.float64)
    elif bad == "f32_out":
        outd["u_re"][0] = torch.zeros(n, dtype=torch.float32, device=DEV)
    elif bad == "missing_im":
        outd["u_im"] = list(out.u_re)
    else:
        states = [torch.empty(n, dtype=torch.float64, device=DEV) for _ in range(5)]
    with pytest.raises(ValueError):
        launch_device(n, ins, None, outd, 0, 0, states)


def test_run_batch_into_rejects_short_device_outputs():
    re, im = synth.generate_device(1, 1, 0, 1024, device=DEV)
    batch = b2s.Batch2x2(n=1024, re=re, im=im)
    out = b2s.SvdBatchOut.empty(1024, True, device=DEV)
    out.smax = out.smax[:512]
    with pytest.raises(ValueError):
        b2s.run_batch_into(batch, out, b2s.RunConfig(field="complex"))


def test_in_process_multi_device_host_shards():
    """RunConfig(devices=(0, 0)): two host threads stream two contiguous
    shards through the host-buffer C-ABI (the reference's thread pool,
    driver.py:180-187); identical trains to one worker and to the oracle."""
    n = 200_003
    for config in (2, 4):
        re, im = synth.generate(config, 9, 0, n)
        batch = b2s.from_trains(re, im)
        field = batch.field
        one, _ = b2s.run_batch(batch, b2s.RunConfig(field=field))
        two, _ = b2s.run_batch(batch, b2s.RunConfig(field=field, devices=(0, 0)))
        three, _ = b2s.run_batch(batch, b2s.RunConfig(field=field, devices=(0, 0, 0), chunk=8192))
        ref = oracle.svd2(batch.re, batch.im)
        for name, arr in ref.trains().items():
            assert_bits_equal(one.trains()[name], arr, "1 worker %s" % name)
            assert_bits_equal(two.trains()[name], arr, "2 workers %s" % name)
            assert_bits_equal(three.trains()[name], arr, "3 workers %s" % name)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_non_current_device_launches_on_the_tensors_device():  # pragma: no cover
    dev1 = torch.device("cuda", 1)
    re, im = synth.generate(1, 2, 0, 4096)
    ref = oracle.svd2(re, im)
    with torch.cuda.device(0):
        got = b2s.svd2_lanes([torch.from_numpy(x).to(dev1) for t in range(4)
                              for x in (re[t], im[t])])
        out, _ = b2s.run_batch(b2s.from_trains(re, im).to(dev1), b2s.RunConfig(field="complex"))
    assert got.smax_scaled.device == dev1
    assert_bits_equal(got.smax_scaled.cpu().numpy(), ref.smax, "svd2_lanes smax")
    assert_bits_equal(out.cpu().smax, ref.smax, "run_batch smax")


@pytest.mark.parametrize("layout", ["pinned", "pageable", "mixed"])
def test_host_path_pinned_and_pageable_trains(layout):
    """The host-buffer C-ABI streams pinned trains directly and bounces
    pageable ones (a lanesvd caller's aligned_zeros arrays) through its own
    pinned buffers; every combination gives the oracle's trains, across
    several pipeline chunks and a ragged last chunk."""
    n = 3 * 65536 + 1000
    for config in (2, 4):
        re, im = synth.generate(config, 12, 0, n)
        cplx = im is not None
        pin = lambda shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
        page = lambda shape: (b2s.aligned_zeros(*shape) if len(shape) == 2
                              else b2s.aligned_zeros(1, shape[0])[0])
        n_hat = b2s.padded_len(n)
        alloc_in = pin if layout in ("pinned", "mixed") else page
        alloc_out = pin if layout == "pinned" else page
        bre = alloc_in((4, n_hat))
        bre[:] = 0.0
        bre[:, :n] = re
        bim = None
        if cplx:
            bim = alloc_in((4, n_hat))
            bim[:] = 0.0
            bim[:, :n] = im
        batch = b2s.Batch2x2(n=n, re=bre, im=bim)
        out = b2s.SvdBatchOut(n=n, u_re=alloc_out((4, n_hat)),
                              u_im=alloc_out((4, n_hat)) if cplx else None,
                              v_re=alloc_out((4, n_hat)),
                              v_im=alloc_out((4, n_hat)) if cplx else None,
                              smax=alloc_out((n_hat,)), smin=alloc_out((n_hat,)),
                              shift=alloc_out((n_hat,)))
        b2s.run_batch_into(batch, out, b2s.RunConfig(field=batch.field, chunk=65536))
        ref = oracle.svd2(batch.re, batch.im)
        for name, arr in ref.trains().items():
            assert_bits_equal(out.trains()[name], arr, "%s %s" % (layout, name))
