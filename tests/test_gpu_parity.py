"""GPU parity: the sm_100a kernels vs the reference, bit for bit.

Every comparison goes through the C-ABI (libb2s.so) via the package's
public API.  Ground truth is the reference's own output (tests/golden/,
made by running lanesvd) and, for arbitrary inputs, the oracle pinned to it.
"""

import os

import numpy as np
import pytest

from helpers import assert_bits_equal, digest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2005_07403_b200 as b2s  # noqa: E402
from paper_2005_07403_b200 import _lib, synth  # noqa: E402
from paper_2005_07403_b200.layout import Batch2x2, from_trains  # noqa: E402
from paper_2005_07403_b200.svd2 import dump_trains  # noqa: E402

DEV = torch.device("cuda", 0)
RECORD_MODES = {"patterned_real_safe": ("safe", False),
                "fuzz_real_safe": ("safe", False),
                "fuzz_real_unc": ("unconditional", False),
                "fuzz_real_sine": ("none", True),
                "fuzz_complex_sine": ("none", True)}


def _dev_batch(re, im):
    b = from_trains(re, im)
    return b.to(DEV)


def _host_digests(out):
    return {k: digest(v.cpu().numpy() if hasattr(v, "cpu") else v)
            for k, v in out.trains().items()}


def test_device_fp_env():
    assert _lib.lib.b2s_check_fp_env(0) == 0


def test_lane_records_device_path(lanes):
    for name, rec in lanes.items():
        mode, sine = RECORD_MODES.get(name, ("none", False))
        re, im = rec["in_re"], rec.get("in_im")
        b = _dev_batch(re, im)
        out, wall = b2s.run_batch(b, b2s.RunConfig(field=b.field, backscale_mode=mode),
                                  sine_form=sine)
        assert wall > 0
        host = out.cpu()
        n = re.shape[1]
        for k, arr in host.trains().items():
            got = arr[..., :n]
            assert_bits_equal(got, rec[k][..., :n], "%s/%s" % (name, k))


def test_lane_records_host_path(lanes):
    for name, rec in lanes.items():
        mode, sine = RECORD_MODES.get(name, ("none", False))
        b = from_trains(rec["in_re"], rec.get("in_im"))
        out, _ = b2s.run_batch(b, b2s.RunConfig(field=b.field, backscale_mode=mode),
                               sine_form=sine)
        n = rec["in_re"].shape[1]
        for k, arr in out.trains().items():
            assert_bits_equal(arr[..., :n], rec[k][..., :n], "%s/%s" % (name, k))


def test_state_dump_matches_reference(lanes):
    for name, rec in lanes.items():
        if "states" not in rec:
            continue
        parts = [rec["in_re"][t] for t in range(4)]
        if "in_im" in rec:
            parts = [x for t in range(4) for x in (rec["in_re"][t], rec["in_im"][t])]
        _, scale, urv, tri = b2s.svd2_lanes(tuple(parts), with_states=True)
        got = np.stack(dump_trains(scale, urv, tri))
        assert_bits_equal(got, rec["states"], name + "/states")


def test_with_states_tuple_matches_reference(lanes):
    """svd2_lanes(with_states=True) returns the reference's
    (Svd2, ScaleResult, UrvState, TriangleSvd) (svd2.py:568-569): every
    field bit-identical to lanesvd's own on the golden lane sets -- the
    dump trains (lanes.npz) and the scaled parts and triangle sec2 / cos
    (states_full.npz, make_states_full.py)."""
    full = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                "states_full.npz"))
    for name, rec in lanes.items():
        if "states" not in rec:
            continue
        parts = [rec["in_re"][t] for t in range(4)]
        if "in_im" in rec:
            parts = [x for t in range(4) for x in (rec["in_re"][t], rec["in_im"][t])]
        svd, scale, urv, tri = b2s.svd2_lanes(tuple(parts), with_states=True)
        assert isinstance(scale, b2s.ScaleResult) and isinstance(urv, b2s.UrvState)
        assert isinstance(tri, b2s.TriangleSvd)
        assert urv.swap_cols.dtype == np.bool_ and len(scale.parts) == len(parts)
        assert (urv.row_phase1[1] is None) == ("in_im" not in rec)
        assert_bits_equal(np.stack(scale.parts), full[name + "/scaled_parts"], name + "/parts")
        assert_bits_equal(np.stack([tri.left_sec2, tri.left_cos, tri.right_sec2, tri.right_cos]),
                          full[name + "/tri"], name + "/tri")
        assert_bits_equal(tri.smax_scaled, svd.smax_scaled, name + "/smax")


@pytest.mark.parametrize("config", [0, 1, 2])
def test_full_config_digests(digests, config):
    entry = digests["configs"][str(config)]
    n = entry["n"]
    re, im = synth.generate_device(config, digests["seed"], 0, n, device=DEV)
    assert digest(re.cpu().numpy()) == entry["input"]["re"], "device synth drifted"
    if im is not None:
        assert digest(im.cpu().numpy()) == entry["input"]["im"]
    b = Batch2x2(n=n, re=re, im=im)
    for key in ("none", "safe", "unconditional", "sine"):
        if key not in entry:
            continue
        mode = key if key in ("safe", "unconditional") else "none"
        out, _ = b2s.run_batch(b, b2s.RunConfig(field=b.field, backscale_mode=mode),
                               sine_form=key == "sine")
        assert _host_digests(out) == entry[key], (config, key)


@pytest.mark.parametrize("config", [3, 4])
def test_large_config_windows(digests, config):
    entry = digests["configs"][str(config)]
    W = digests["window"]
    for w in entry["windows"]:
        re, im = synth.generate_device(config, digests["seed"], w["lo"], W, device=DEV)
        assert digest(re.cpu().numpy()) == w["input"]["re"]
        out, _ = b2s.run_batch(Batch2x2(n=W, re=re, im=im),
                               b2s.RunConfig(field="real" if im is None else "complex"))
        assert _host_digests(out) == w["none"], (config, w["lo"])


@pytest.mark.parametrize("config", [0, 1, 2, 3, 4])
def test_device_synth_equals_host_synth(config):
    for lo, n in ((0, 4096), (123456, 1000), (5, 77)):
        hr, hi = synth.generate(config, 99, lo, n)
        dr, di = synth.generate_device(config, 99, lo, n, device=DEV)
        assert_bits_equal(dr.cpu().numpy(), hr, "re")
        if hi is not None:
            assert_bits_equal(di.cpu().numpy(), hi, "im")


@pytest.mark.parametrize("field", ["real", "complex"])
def test_fuzz_vs_oracle_1m(field):
    rng = np.random.default_rng(11)
    k = 8 if field == "complex" else 4
    n = 1 << 20
    v = rng.integers(0, 2 ** 64, size=(k, n), dtype=np.uint64).view(np.float64).copy()
    v[~np.isfinite(v)] = 1.0
    v[rng.random((k, n)) < 0.1] = 0.0
    re, im = (v[0::2], v[1::2]) if field == "complex" else (v, None)
    ref = oracle.svd2(re, im)
    out, _ = b2s.run_batch(_dev_batch(re, im), b2s.RunConfig(field=field))
    host = out.cpu()
    for name, arr in ref.trains().items():
        assert_bits_equal(host.trains()[name], arr, name)


def test_backscale_kernel_vs_oracle():
    rng = np.random.default_rng(5)
    n = 1 << 16
    smax = np.abs(rng.standard_normal(n)) * np.exp2(rng.integers(-1074, 1023, n))
    smin = smax * rng.random(n)
    smin[::7] = 0.0
    shift = rng.integers(-2, 2096, n).astype(np.float64)
    shift[::11] = 1.7976931348623157e308
    for mode in ("none", "safe", "unconditional"):
        ref = oracle.backscale(smax, smin, shift, mode)
        got = b2s.backscale(smax, smin, shift, mode)
        for r, g in zip(ref, got):
            assert_bits_equal(g, r, mode)


def test_partition_and_shard_invariance():
    re, _ = synth.generate_device(3, 1, 0, 1 << 20, device=DEV)
    b = Batch2x2(n=1 << 20, re=re)
    whole, _ = b2s.run_batch(b, b2s.RunConfig())
    lo = Batch2x2(n=1 << 19, re=re[:, : 1 << 19].contiguous())
    hi = Batch2x2(n=1 << 19, re=re[:, 1 << 19:].contiguous())
    a, _ = b2s.run_batch(lo, b2s.RunConfig())
    c, _ = b2s.run_batch(hi, b2s.RunConfig())
    assert torch.equal(torch.cat([a.u_re, c.u_re], 1).view(torch.int64), whole.u_re.view(torch.int64))
    assert torch.equal(torch.cat([a.smax, c.smax]).view(torch.int64), whole.smax.view(torch.int64))


def test_repeat_determinism():
    re, im = synth.generate_device(4, 2, 0, 1 << 18, device=DEV)
    b = Batch2x2(n=1 << 18, re=re, im=im)
    a, _ = b2s.run_batch(b, b2s.RunConfig(field="complex"))
    c, _ = b2s.run_batch(b, b2s.RunConfig(field="complex"))
    for k in a.trains():
        assert torch.equal(a.trains()[k].view(torch.int64), c.trains()[k].view(torch.int64))


def test_host_pipeline_chunks_equal_device():
    n = 300_000
    re, im = synth.generate(1, 4, 0, n)
    b = from_trains(re, im)
    ref = oracle.svd2(b.re, b.im)
    for chunk in (0, 4096, 65536 + 8):
        out, _ = b2s.run_batch(b, b2s.RunConfig(field="complex", chunk=chunk))
        for k, arr in ref.trains().items():
            assert_bits_equal(out.trains()[k], arr, "%s chunk=%d" % (k, chunk))


def test_chunk_and_single_entry_points():
    re = np.zeros((4, 8))
    re[0] = 1.0
    re[3] = 1.0
    res = b2s.svd2_chunk(re)
    assert (res.shift == 1021.0).all() and (res.smax == 2.0 ** 1021).all()
    a = np.array([[1 + 1j, 0], [0, 2 - 1j]])
    one = b2s.svd2_single(a)
    assert one.u.dtype == np.complex128
    s = np.array([one.smax, one.smin]) * 2.0 ** -one.shift
    rec = one.u @ np.diag(s) @ one.v.conj().T
    assert np.abs(rec - a).max() < 1e-15 * np.abs(a).max()


def test_padding_lanes_and_empty_batch():
    b = b2s.pack(np.random.default_rng(1).standard_normal((5, 2, 2)))
    out, _ = b2s.run_batch(b, b2s.RunConfig())
    assert (out.smax[5:] == 0.0).all()
    assert (out.shift[5:] == 1.7976931348623157e308).all()
    empty = b2s.pack(np.zeros((0, 2, 2)))
    out, wall = b2s.run_batch(empty, b2s.RunConfig())
    assert out.n == 0 and out.n_hat == 0


def test_invalid_arguments_raise_valueerror():
    b = b2s.pack(np.eye(2).reshape(1, 2, 2))
    with pytest.raises(ValueError):
        b2s.run_batch(b, b2s.RunConfig(field="complex"))
    with pytest.raises(TypeError):
        b2s.run_batch(b.re, b2s.RunConfig())
    with pytest.raises(ValueError):
        b2s.svd2_lanes((np.zeros(3), np.zeros(3)))
    with pytest.raises(ValueError):
        b2s.backscale(np.ones(1), np.ones(1), np.zeros(1), mode="maybe")


def test_hard_lane_queue_counts():
    """Moderate-exponent configs take the fast path on (nearly) every lane;
    config 2 (full exponent range, structured zeros) queues many lanes for
    the exact fix-up -- results are bit-identical either way (digest tests)."""
    for config, n, bound in ((3, 1 << 20, 1e-3), (1, 1 << 20, 1e-3), (2, 1 << 20, 1.0)):
        re, im = synth.generate_device(config, 5, 0, n, device=DEV)
        b2s.run_batch(Batch2x2(n=n, re=re, im=im),
                      b2s.RunConfig(field="real" if im is None else "complex"))
        c = _lib.lib.b2s_hard_lane_count(0)
        assert 0 <= c <= bound * n, (config, c)
        print("config %d: %d hard lanes of %d" % (config, c, n))


@pytest.mark.parametrize("field,n", [("real", 300_005), ("complex", 77_777), ("real", 8), ("complex", 1 << 16)])
def test_record_ingest_equals_trains(field, n):
    """Direct AoSoA-8 ingest (TMA blocks of 32 records) == SoA trains."""
    from paper_2005_07403_b200 import records as R
    rng = np.random.default_rng(n)
    k = 8 if field == "complex" else 4
    v = rng.integers(0, 2 ** 64, size=(k, n), dtype=np.uint64).view(np.float64).copy()
    v[~np.isfinite(v)] = 0.5
    re, im = (v[0::2], v[1::2]) if field == "complex" else (v, None)
    recs = R.trains_to_records(re, im)
    out = R.run_records(recs, n, field).cpu()
    ref = oracle.svd2(b2s.from_trains(re, im).re, b2s.from_trains(re, im).im)
    for name, arr in ref.trains().items():
        assert_bits_equal(out.trains()[name], arr, name)


def test_misaligned_trains_take_ldg_path():
    """Trains only 8-byte aligned (odd lane offset) cannot feed the TMA ring;
    the register-prefetch kernels run instead, with identical results."""
    n = 50_001
    re, im = synth.generate_device(1, 3, 0, n + 1, device=DEV)
    re_v = [re[t][1:] for t in range(4)]          # 8-byte aligned views
    im_v = [im[t][1:] for t in range(4)]
    assert re_v[0].data_ptr() % 16 == 8
    out = b2s.SvdBatchOut.empty(n, True, device=DEV)
    outd = {"u_re": list(out.u_re), "u_im": list(out.u_im), "v_re": list(out.v_re),
            "v_im": list(out.v_im), "smax": out.smax, "smin": out.smin, "shift": out.shift}
    from paper_2005_07403_b200.svd2 import launch_device
    launch_device(n, re_v, im_v, outd, 0)
    torch.cuda.synchronize()
    ref = oracle.svd2(re[:, 1:].cpu().numpy(), im[:, 1:].cpu().numpy())
    host = out.cpu()
    for name, arr in ref.trains().items():
        assert_bits_equal(host.trains()[name][..., :n], arr, name)


def test_nonfinite_inputs_do_not_hang():
    """Non-finite entries are rejected at ingest (pack / from_trains, as in
    layout.py:133-186); fed raw to the kernels they must still terminate."""
    re = torch.tensor([[np.nan, np.inf, -np.inf, 1.0, 0.0, 1.0, 5e-324, 1e308]] * 4,
                      dtype=torch.float64, device=DEV)
    out, _ = b2s.run_batch(Batch2x2(n=8, re=re), b2s.RunConfig())
    torch.cuda.synchronize()
    assert out.smax.shape == (8,)
    with pytest.raises(ValueError):
        b2s.pack(np.full((1, 2, 2), np.nan))


def test_sub_launch_boundaries_small_chunk_host_path():
    """Host pipeline chunk edges at arbitrary positions (ragged tails)."""
    n = 10_007
    re, _ = synth.generate(2, 8, 0, n)
    b = from_trains(re)
    ref = oracle.svd2(b.re)
    for chunk in (256, 1000, 4096):
        out, _ = b2s.run_batch(b, b2s.RunConfig(chunk=chunk))
        for k, arr in ref.trains().items():
            assert_bits_equal(out.trains()[k], arr, "%s chunk=%d" % (k, chunk))


def _outd(out):
    return {"u_re": list(out.u_re), "v_re": list(out.v_re),
            "u_im": None if out.u_im is None else list(out.u_im),
            "v_im": None if out.v_im is None else list(out.v_im),
            "smax": out.smax, "smin": out.smin, "shift": out.shift}


def _launch(re, im, out, stream):
    from paper_2005_07403_b200.svd2 import launch_device
    launch_device(re.shape[1], list(re), None if im is None else list(im), _outd(out), 0,
                  stream=stream.cuda_stream)


def test_concurrent_streams_keep_separate_hard_lane_queues():
    """Launches on different streams run concurrently, each with its own
    hard-lane mask and counter (config 4 has fix-up lanes): the results of
    interleaved launches equal those of sequential ones."""
    n = 1 << 19
    batches = [synth.generate_device(4, 11 + k, k * n, n, device=DEV) for k in range(4)]
    ref = []
    for re, im in batches:
        out = b2s.SvdBatchOut.empty(n, True, device=DEV)
        _launch(re, im, out, torch.cuda.current_stream())
        torch.cuda.synchronize()
        ref.append(out.cpu())
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [b2s.SvdBatchOut.empty(n, True, device=DEV) for _ in batches]
    torch.cuda.synchronize()
    for rep in range(3):
        for k, (re, im) in enumerate(batches):
            _launch(re, im, outs[k], streams[k % 2])
    torch.cuda.synchronize()
    for k in range(len(batches)):
        got = outs[k].cpu().trains()
        for name, arr in ref[k].trains().items():
            assert_bits_equal(got[name], arr, "batch %d %s" % (k, name))


def test_cuda_graph_capture_after_reserve():
    """With the stream's workspace reserved, a launch can be captured into a
    CUDA graph and replayed (no allocation during capture)."""
    n = 1 << 18
    re, im = synth.generate_device(4, 3, 0, n, device=DEV)
    ref = b2s.SvdBatchOut.empty(n, True, device=DEV)
    _launch(re, im, ref, torch.cuda.current_stream())
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    assert _lib.lib.b2s_reserve_workspace(0, n, s.cuda_stream) == 0
    out = b2s.SvdBatchOut.empty(n, True, device=DEV)
    with torch.cuda.stream(s):
        _launch(re, im, out, s)                      # warm-up on the capture stream
    torch.cuda.synchronize()
    for name in ("smax", "smin", "shift"):
        getattr(out, name).zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        _launch(re, im, out, s)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    got, want = out.cpu().trains(), ref.cpu().trains()
    for name, arr in want.items():
        assert_bits_equal(got[name], arr, name)


@pytest.mark.parametrize("config", [2, 4])
@pytest.mark.parametrize("path", ["records", "misaligned", "sine", "safe"])
def test_stress_configs_every_kernel_path(config, path):
    """The full-range (2) and mixed wide-exponent (4) configs through every
    kernel variant -- AoSoA-8 records on the TMA ring, the register-prefetch
    kernels (8-byte-aligned views), the sine-form assembly and the safe
    backscale epilogue -- bit-identical to the oracle."""
    from paper_2005_07403_b200 import records as R
    from paper_2005_07403_b200.svd2 import launch_device
    n = 40_000 + 8 * config
    re, im = synth.generate(config, 17, 1000, n + 8)
    mode = "safe" if path == "safe" else "none"
    sine = path == "sine"
    if path == "records":
        out = R.run_records(R.trains_to_records(re[:, :n], None if im is None else im[:, :n]), n,
                            "complex" if im is not None else "real").cpu()
        got = {k: v[..., :n] for k, v in out.trains().items()}
    elif path == "misaligned":
        dre = torch.from_numpy(np.ascontiguousarray(re)).to(DEV)
        dim = None if im is None else torch.from_numpy(np.ascontiguousarray(im)).to(DEV)
        out = b2s.SvdBatchOut.empty(n, im is not None, device=DEV)
        launch_device(n, [dre[t][1:n + 1] for t in range(4)],
                      None if dim is None else [dim[t][1:n + 1] for t in range(4)], _outd(out), 0)
        torch.cuda.synchronize()
        got = {k: v[..., :n] for k, v in out.cpu().trains().items()}
        re, im = re[:, 1:n + 1], None if im is None else im[:, 1:n + 1]
    else:
        b = from_trains(re[:, :n], None if im is None else im[:, :n]).to(DEV)
        out, _ = b2s.run_batch(b, b2s.RunConfig(field=b.field, backscale_mode=mode), sine_form=sine)
        got = {k: v[..., :n] for k, v in out.cpu().trains().items()}
    ref = oracle.svd2(np.ascontiguousarray(re[:, :n]), None if im is None else np.ascontiguousarray(im[:, :n]),
                      backscale_mode=mode, sine_form=sine)
    for name, arr in ref.trains().items():
        assert_bits_equal(got[name], arr[..., :n], "config %d %s %s" % (config, path, name))


_SUBLAUNCH_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import oracle, paper_2005_07403_b200 as b2s
from paper_2005_07403_b200 import synth, records as R
from paper_2005_07403_b200.layout import from_trains
n = 3 * 65536 + 1000
for config in (2, 4):
    re, im = synth.generate(config, 23, 5000, n)
    ref = oracle.svd2(re, im).trains()
    b = from_trains(re, im).to("cuda")
    out, _ = b2s.run_batch(b, b2s.RunConfig(field=b.field))
    rec = R.run_records(R.trains_to_records(re, im), n, b.field).cpu().trains()
    for name, got in (("trains", out.cpu().trains()), ("records", rec)):
        for k, arr in ref.items():
            g = np.ascontiguousarray(got[k][..., :n]).view(np.uint64)
            if not np.array_equal(g, np.ascontiguousarray(arr).view(np.uint64)):
                print("MISMATCH config %d %s %s" % (config, name, k)); sys.exit(1)
print("OK")
"""


def test_sub_launch_split_on_device():
    """Device batches larger than one sub-launch (B2S_MAX_LAUNCH forces
    65 536-lane sub-launches: 3 full ones and a ragged fourth with a
    sub-tile tail) through the SoA and AoSoA-8 kernels, configs 2 and 4
    (fix-up lanes in several sub-launches): bit-identical to the oracle."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, B2S_MAX_LAUNCH="65536")
    r = subprocess.run([sys.executable, "-c", _SUBLAUNCH_SCRIPT, root], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr


def _random_finite(rng, count):
    """Uniform 64-bit patterns with non-finite ones redrawn: the whole
    magnitude range, subnormals and both zero signs (the fuzz corpus of the
    reference's acceptance suite, test_acceptance.py:70-101)."""
    vals = rng.integers(0, 2 ** 64, size=count, dtype=np.uint64).view(np.float64)
    bad = ~np.isfinite(vals)
    while bad.any():
        vals[bad] = rng.integers(0, 2 ** 64, size=int(bad.sum()), dtype=np.uint64).view(np.float64)
        bad = ~np.isfinite(vals)
    return vals


@pytest.mark.parametrize("field", ["real", "complex"])
def test_theorem1_invariants_full_range_fuzz(field):
    """test_acceptance.py:115-140 on 2^20 full-bit-pattern lanes per field:
    scaled singular values finite, sorted and non-negative; |tan psi| <=
    sqrt(2)(1 + 2 eps53); |tan psi| >= |tan phi|; cos psi >= (1 - 2 eps53)
    / sqrt(3); every factor finite -- on the streaming kernels' outputs and
    the state dump, which must agree bit for bit."""
    eps = 2.0 ** -53
    n = 1 << 20
    rng = np.random.default_rng(2026 if field == "real" else 2027)
    ntr = 4 if field == "real" else 8
    parts = tuple(torch.from_numpy(_random_finite(rng, n)).to(DEV) for _ in range(ntr))
    svd, _scale, urv, tri = b2s.svd2_lanes(parts, with_states=True)
    re = torch.stack(parts[0::2] if ntr == 8 else parts)
    im = torch.stack(parts[1::2]) if ntr == 8 else None
    fast, _ = b2s.run_batch(b2s.Batch2x2(n=n, re=re, im=im), b2s.RunConfig(field=field))
    smax, smin = fast.smax.cpu().numpy(), fast.smin.cpu().numpy()
    assert_bits_equal(smax, svd.smax_scaled.cpu().numpy(), "smax fast vs state-dump kernel")
    assert_bits_equal(smin, svd.smin_scaled.cpu().numpy(), "smin fast vs state-dump kernel")
    assert np.isfinite(smax).all() and np.isfinite(smin).all()
    assert (smax >= smin).all() and (smin >= 0.0).all()
    lt = tri.left_tan.cpu().numpy()
    rt = tri.right_tan.cpu().numpy()
    assert (np.abs(rt) <= np.sqrt(2.0) * (1 + 2 * eps)).all()
    assert (np.abs(rt) >= np.abs(lt)).all()
    # cos psi is V's (1,1) entry before the column swap (svd2.py:350-369)
    swap_c = urv.swap_cols.cpu().numpy()
    v11, v21 = np.abs(svd.v11[0].cpu().numpy()), np.abs(svd.v21[0].cpu().numpy())
    rc = np.where(swap_c, v21, v11)
    assert (rc >= (1 / np.sqrt(3.0)) * (1 - 2 * eps)).all()
    for t in list(fast.u_re) + list(fast.v_re) + ([] if im is None else list(fast.u_im) + list(fast.v_im)):
        assert torch.isfinite(t).all()
