"""Host-side logic (no GPU): layout containers, config validation, sharding,
synthetic inputs, and the C-ABI library surface.

Mirrors the reference's test_layout.py / test_driver.py cases that do not
decompose anything (those run on the GPU in test_gpu_parity.py).
"""

import ctypes
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2005_07403_b200 as b2s
from paper_2005_07403_b200 import _lib, layout, synth
from paper_2005_07403_b200.driver import RunConfig, shards

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------------------
# layout (reference test_layout.py)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n,expect", [(0, 0), (1, 8), (5, 8), (8, 8),
                                      (9, 16), (16, 16), (4097, 4104)])
def test_padded_len_examples(n, expect):
    assert b2s.padded_len(n) == expect


@settings(max_examples=200, deadline=None)
@given(st.integers(min_value=0, max_value=10 ** 9))
def test_padded_len_properties(n):
    p = b2s.padded_len(n)
    assert p % 8 == 0 and n <= p < n + 8


def test_padded_len_rejects_negative():
    with pytest.raises(ValueError):
        b2s.padded_len(-1)


def test_aligned_zeros():
    a = b2s.aligned_zeros(4, 1024)
    assert a.ctypes.data % 64 == 0 and a.flags.c_contiguous
    assert a.dtype == np.float64 and not a.any()
    with pytest.raises(ValueError):
        b2s.aligned_zeros(4, 12)


def test_pack_real_layout_and_padding():
    mats = np.arange(20, dtype=np.float64).reshape(5, 2, 2)
    b = b2s.pack(mats)
    assert b.n == 5 and b.n_hat == 8 and b.field == "real"
    assert b.re.ctypes.data % 64 == 0
    # column-major entry order e11, e21, e12, e22
    assert b.re[:, 1].tolist() == [4.0, 6.0, 5.0, 7.0]
    assert (b.re[:, 5:] == 0).all()


def test_pack_complex_placement():
    mats = np.array([[[1 + 2j, 3 - 4j], [5 + 0j, -6j]]])
    b = b2s.pack(mats)
    assert b.field == "complex"
    assert b.re[:, 0].tolist() == [1.0, 5.0, 3.0, 0.0]
    assert b.im[:, 0].tolist() == [2.0, 0.0, -4.0, -6.0]


@pytest.mark.parametrize("bad", [np.inf, -np.inf, np.nan])
def test_pack_rejects_nonfinite(bad):
    mats = np.ones((3, 2, 2))
    mats[1, 0, 1] = bad
    with pytest.raises(ValueError):
        b2s.pack(mats)
    with pytest.raises(ValueError):
        b2s.pack(mats.astype(np.complex128))


def test_pack_unpack_inputs_roundtrip_bits():
    rng = np.random.default_rng(1)
    bitsv = rng.integers(0, 2 ** 64, size=(37, 2, 2), dtype=np.uint64)
    mats = bitsv.view(np.float64).copy()
    mats[~np.isfinite(mats)] = -0.0
    mats[0, 0, 0] = 5e-324
    back = b2s.unpack_inputs(b2s.pack(mats))
    assert np.array_equal(back.view(np.uint64), mats.view(np.uint64))
    c = mats + 1j * mats[:, ::-1, :]
    cb = b2s.unpack_inputs(b2s.pack(c))
    assert np.array_equal(cb.view(np.uint64), c.view(np.uint64))


def test_from_trains_and_shape_checks():
    re = np.arange(12, dtype=np.float64).reshape(4, 3)
    b = b2s.from_trains(re)
    assert b.n == 3 and b.n_hat == 8
    with pytest.raises(ValueError):
        b2s.from_trains(np.zeros((3, 8)))
    with pytest.raises(ValueError):
        b2s.from_trains(np.zeros((4, 8)), np.zeros((4, 9)))
    with pytest.raises(ValueError):
        b2s.Batch2x2(n=3, re=np.zeros((4, 12)))
    with pytest.raises(ValueError):
        b2s.Batch2x2(n=9, re=np.zeros((4, 8)))


def test_unpack_records():
    out = b2s.SvdBatchOut.empty(3, complex_field=False)
    out.u_re[0, :] = 1.0
    out.smax[:] = [1.0, 2.0, 3.0, 0, 0, 0, 0, 0]
    recs = b2s.unpack(out)
    assert len(recs) == 3 and recs[2].smax == 3.0
    assert recs[0].u[0, 0] == 1.0 and recs[0].u.shape == (2, 2)


# ---------------------------------------------------------------------------
# RunConfig and sharding (reference test_driver.py:41-65)
# ---------------------------------------------------------------------------

def test_config_defaults():
    cfg = RunConfig()
    assert cfg.field == "real" and cfg.path == "cuda" and cfg.backscale_mode == "none"


@pytest.mark.parametrize("kw", [dict(field="rational"), dict(path="simd"),
                                dict(threads=-1), dict(backscale_mode="maybe"),
                                dict(devices=()), dict(devices=(-1,)),
                                dict(chunk=-5)])
def test_config_rejects_bad_values(kw):
    with pytest.raises(ValueError):
        RunConfig(**kw)


def test_reference_path_names_accepted():
    for p in ("vectorized", "pointwise", "cuda"):
        assert RunConfig(path=p).path == p


@pytest.mark.parametrize("n_hat", [8, 64, 1024, 4096, 100008, 1 << 30])
@pytest.mark.parametrize("parts", [1, 2, 3, 7, 8, 16])
def test_shards_cover_and_align(n_hat, parts):
    spans = shards(n_hat, parts)
    assert spans[0][0] == 0 and spans[-1][1] == n_hat
    for (lo, hi), (lo2, _) in zip(spans, spans[1:]):
        assert hi == lo2 and lo % 256 == 0
    assert len(spans) <= parts
    if n_hat >= 256 * parts:
        sizes = [hi - lo for lo, hi in spans]
        assert len(spans) == parts and max(sizes) - min(sizes) <= 512


def test_shards_empty():
    assert shards(0, 4) == []


def test_run_batch_type_and_field_errors_before_any_gpu_work():
    b = b2s.pack(np.eye(2).reshape(1, 2, 2))
    with pytest.raises(TypeError):
        b2s.run_batch(b.re, RunConfig())
    with pytest.raises(ValueError):
        b2s.run_batch(b, RunConfig(field="complex"))


# ---------------------------------------------------------------------------
# synthetic inputs (host side of the counter-based generator)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("config", [0, 1, 2, 3, 4])
def test_synth_shard_consistency(config):
    whole_re, whole_im = synth.generate(config, 9, 1000, 3000)
    a_re, a_im = synth.generate(config, 9, 1000, 1234)
    b_re, b_im = synth.generate(config, 9, 2234, 1766)
    assert np.array_equal(np.concatenate([a_re, b_re], 1).view(np.uint64),
                          whole_re.view(np.uint64))
    if whole_im is not None:
        assert np.array_equal(np.concatenate([a_im, b_im], 1).view(np.uint64),
                              whole_im.view(np.uint64))
    vals = whole_re if whole_im is None else np.concatenate([whole_re, whole_im])
    assert np.isfinite(vals).all()


def test_synth_distributions():
    re, _ = synth.generate(0, 3, 0, 1 << 16)
    e = np.frexp(re)[1] - 1
    assert e.min() == -20 and e.max() == 20
    m = np.abs(re) / np.exp2(e)
    assert (m >= 1).all() and (m < 2).all()
    re2, _ = synth.generate(2, 3, 0, 1 << 16)
    nz = re2[re2 != 0]
    assert (np.abs(nz) < 2.0 ** -1022).any()          # subnormals present
    cls, _ = synth.lane_class(3, 2, np.arange(1 << 16, dtype=np.uint64))
    frac = np.bincount(cls, minlength=10) / (1 << 16)
    assert np.allclose(frac, 0.1, atol=0.01)
    # diagonal lanes have zero off-diagonals
    assert (re2[1, cls == 2] == 0).all() and (re2[2, cls == 2] == 0).all()
    re4, im4 = synth.generate(4, 3, 0, 1 << 14)
    cls4, _ = synth.lane_class(3, 4, np.arange(1 << 14, dtype=np.uint64))
    tri = (cls4 == 6) | (cls4 == 7)
    assert (re4[1, tri] == 0).all() and (im4[1, tri] == 0).all()


def test_make_value_subnormal_rounding():
    # mantissa 1 + k 2^-52 at exponent -1074 rounds to 2^-1074 or 2^-1073
    sm = np.array([0, (1 << 51), (1 << 51) + 1, (1 << 52) - 1], dtype=np.uint64)
    v = synth.make_value(sm, np.full(4, -1074))
    assert v.view(np.uint64).tolist() == [1, 2, 2, 2]
    v = synth.make_value(np.array([1 << 63], dtype=np.uint64), np.array([5]))
    assert v[0] == -32.0


# ---------------------------------------------------------------------------
# C-ABI surface: the library loads and exports every declared symbol
# ---------------------------------------------------------------------------

def _declared_symbols():
    with open(os.path.join(REPO, "include", "b2s.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(b2s_[a-z0-9_]+)\s*\(", text)))


def _exported_symbols(path):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True,
                         text=True, check=True).stdout
    return sorted({ln.split()[-1] for ln in out.splitlines()
                   if ln.split() and ln.split()[-1].startswith("b2s_")})


def test_header_and_library_agree():
    """Both directions: every function include/b2s.h declares is exported,
    and the library exports no b2s_ symbol the header does not declare
    (diagnostic probes live only in the tools build, -DB2S_DIAGNOSTICS)."""
    declared = _declared_symbols()
    assert set(declared) == set(_lib.SYMBOLS)
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(raw, name), name
    assert _exported_symbols(_lib.LIB_PATH) == declared
    assert _lib.lib.b2s_version() >= 100


def test_lazy_library_maps_on_first_error_check():
    """_lib.check() is the first native call of many paths (an argument
    error before any other call): it must map the library itself."""
    import subprocess
    import sys
    code = ("from paper_2005_07403_b200 import _lib\n"
            "try:\n    _lib.check(3, 'x')\nexcept ValueError:\n    pass\n"
            "assert _lib.loaded()\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       cwd=REPO, timeout=300)
    assert r.returncode == 0, r.stderr


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_capi_argument_validation_without_gpu():
    """Invalid arguments are rejected (rc > 0, message set) before any CUDA
    call, mirroring the reference's ValueError paths."""
    L = _lib.lib
    rc = L.b2s_svd2_real(-1, None, None, None, None, None, None, 0, 0, None, None)
    assert rc > 0 and b"negative" in L.b2s_last_error()
    arr, _keep = _lib.ptr_array([8, 8, 8, 8])
    rc = L.b2s_svd2_real(4, arr, arr, arr, 8, 8, 8, 7, 0, None, None)
    assert rc > 0 and b"backscale_mode" in L.b2s_last_error()
    rc = L.b2s_svd2_complex(4, arr, arr, arr, arr, arr, arr, 8, 8, 8, 0, 64, None, None)
    assert rc > 0 and b"flag" in L.b2s_last_error()
    rc = L.b2s_svd2_real(4, arr, arr, arr, 8, 8, 8, 0, 2, None, None)
    assert rc > 0 and b"states" in L.b2s_last_error()
    bad, _k2 = _lib.ptr_array([8, 8, 12, 8])
    rc = L.b2s_svd2_real(4, bad, arr, arr, 8, 8, 8, 0, 0, None, None)
    assert rc > 0 and b"aligned" in L.b2s_last_error()
    assert L.b2s_synth(9, 0, 0, 1, arr, None, None) > 0
    assert L.b2s_backscale(1, 8, 8, 8, 5, 8, 8, 8, None) > 0
    assert L.b2s_math_probe(99, 1, 8, 8, 8, None) > 0
    # zero lanes is a valid no-op
    assert L.b2s_svd2_real(0, arr, arr, arr, 8, 8, 8, 0, 0, None, None) == 0
    # the phase, lane-op and reference-SVD entries validate before any CUDA call
    rc = L.b2s_svd2_phase(99, 0, 0, 4, 4, arr, 5, arr, None)
    assert rc > 0 and b"unknown phase" in L.b2s_last_error()
    rc = L.b2s_svd2_phase(0, 0, 0, 4, 4, arr, 4, arr, None)          # compute_scale real: 4 -> 5
    assert rc > 0 and b"takes 4 input and 5 output" in L.b2s_last_error()
    assert L.b2s_svd2_phase(0, 1, 0, -1, 8, arr, 9, arr, None) > 0
    rc = L.b2s_lane_op(77, 4, 1, arr, 1, arr, None)
    assert rc > 0 and b"unknown lane op" in L.b2s_last_error()
    rc = L.b2s_lane_op(0, 4, 2, arr, 1, arr, None)                     # fma takes 3 inputs
    assert rc > 0 and b"takes 3 input" in L.b2s_last_error()
    assert L.b2s_oracle_svd2(4, None, None, arr, None) > 0
    with pytest.raises(ValueError):
        _lib.check(1, "x")
    with pytest.raises(RuntimeError):
        _lib.check(-2, "x")


def test_product_never_imports_oracle():
    """The CUDA product path must not route through the CPU oracle."""
    pkg = os.path.join(REPO, "paper_2005_07403_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


# ---------------------------------------------------------------------------
# Caller-owned buffers are validated before their raw pointers reach the ABI
# ---------------------------------------------------------------------------

def _host_batch_and_out(n=16, cplx=False):
    from paper_2005_07403_b200 import SvdBatchOut
    rng = np.random.default_rng(1)
    re = rng.standard_normal((4, n))
    im = rng.standard_normal((4, n)) if cplx else None
    return b2s.from_trains(re, im), SvdBatchOut.empty(n, cplx)


@pytest.mark.parametrize("bad", ["f32", "short", "strided", "readonly", "list"])
def test_run_batch_into_rejects_bad_host_outputs(bad):
    batch, out = _host_batch_and_out()
    if bad == "f32":
        out.u_re = out.u_re.astype(np.float32)
    elif bad == "short":
        out.smax = out.smax[:8]
    elif bad == "strided":
        out.v_re = np.zeros((4, 2 * batch.n_hat))[:, ::2]
    elif bad == "readonly":
        out.shift.flags.writeable = False
    else:
        out.smin = list(out.smin)
    with pytest.raises(ValueError):
        b2s.run_batch_into(batch, out, b2s.RunConfig())


def test_device_train_check_rejects_host_tensors():
    import torch
    from paper_2005_07403_b200.svd2 import check_device_trains
    with pytest.raises(ValueError, match="CUDA tensor"):
        check_device_trains([torch.zeros(8, dtype=torch.float64)], 8,
                            torch.device("cpu"), "in_re")
