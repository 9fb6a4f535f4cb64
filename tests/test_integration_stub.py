"""INTEGRATION.md's ctypes stub (the binding a lanesvd maintainer adds to
driver.py) is executed as written, against this build of libb2s.so.

CPU: the stub loads the library, its argtypes match the C-ABI, and a call
without a GPU surfaces as RuntimeError (rc < 0), a bad backscale mode as
ValueError (rc > 0).  GPU: the stub decomposes a batch bit-identically to
the oracle (the reference pipeline restated)."""

import os
import re

import numpy as np
import pytest

from paper_2005_07403_b200 import _lib, synth
import paper_2005_07403_b200 as b2s

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as fh:
        text = fh.read()
    code = re.findall(r"```python\n(.*?)```", text, re.S)[0]
    assert "/path/to/paper_2005_07403_b200/_native/libb2s.so" in code
    code = code.replace("/path/to/paper_2005_07403_b200/_native/libb2s.so", _lib.LIB_PATH)
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def _batch(config, n):
    re_, im = synth.generate(config, 3, 0, n)
    batch = b2s.from_trains(re_, im)
    return batch, b2s.SvdBatchOut.empty(batch.n, im is not None)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.mark.skipif(_has_gpu(), reason="CPU-only behaviour")
def test_stub_loads_and_maps_errors_without_gpu():
    ns = _stub()
    assert "cuda" in ns["PATHS"]
    batch, out = _batch(0, 64)
    with pytest.raises(RuntimeError):
        ns["_run_cuda"](batch, out, False, "none")
    L = ns["_lib"]()
    rc = L.b2s_svd2_real_host(8, ns["_rows"](batch.re), ns["_rows"](out.u_re),
                              ns["_rows"](out.v_re), out.smax.ctypes.data, out.smin.ctypes.data,
                              out.shift.ctypes.data, 9, 0, 0, 0)
    assert rc > 0 and b"backscale" in L.b2s_last_error()


@pytest.mark.gpu
@pytest.mark.parametrize("config", [1, 2])
def test_stub_decomposes_like_the_oracle(config):
    if not _has_gpu():  # pragma: no cover
        pytest.skip("no CUDA device")
    import oracle
    from helpers import assert_bits_equal
    ns = _stub()
    batch, out = _batch(config, 100_003)
    ns["_run_cuda"](batch, out, False, "none")
    ref = oracle.svd2(batch.re, batch.im)
    for name, arr in ref.trains().items():
        assert_bits_equal(out.trains()[name], arr, name)
