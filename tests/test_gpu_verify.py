"""GPU double-double verifier (b2s_metrics) vs the reference's own
verify.metrics values (tests/golden/metrics.json, made by running lanesvd)."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

mpmath = pytest.importorskip("mpmath")

import paper_2005_07403_b200 as b2s  # noqa: E402
from paper_2005_07403_b200 import synth  # noqa: E402
from paper_2005_07403_b200.verify import lane_metrics, metrics  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def ref_metrics():
    with open(os.path.join(GOLDEN, "metrics.json")) as fh:
        return json.load(fh)


def _s(x):
    with mpmath.workprec(240):
        return mpmath.nstr(x, 80)


def _check(m, ref, what):
    for k in ("kappa", "rho", "delta", "eta"):
        assert _s(getattr(m, k)) == ref[k], (what, k, _s(getattr(m, k)), ref[k])
    assert m.rho_excluded_lanes == ref["excluded"], what


def test_metrics_on_reference_outputs(lanes, ref_metrics):
    for name, ref in ref_metrics.items():
        if name.endswith("_full"):
            continue
        rec = lanes[name]
        b = b2s.from_trains(rec["in_re"], rec.get("in_im"))
        out = b2s.SvdBatchOut(n=b.n, u_re=rec["u_re"], u_im=rec.get("u_im"), v_re=rec["v_re"],
                              v_im=rec.get("v_im"), smax=rec["smax"], smin=rec["smin"],
                              shift=rec["shift"])
        _check(metrics(b, out), ref, name)


@pytest.mark.parametrize("config", [0, 1])
def test_metrics_on_gpu_outputs_full_config(digests, ref_metrics, config):
    n = digests["configs"][str(config)]["n"]
    re, im = synth.generate_device(config, digests["seed"], 0, n, device="cuda")
    b = b2s.Batch2x2(n=n, re=re, im=im)
    out, _ = b2s.run_batch(b, b2s.RunConfig(field=b.field))
    _check(metrics(b, out), ref_metrics["config%d_full" % config], "config%d" % config)


def test_tolerance_gate_at_scale():
    """North-star tolerances on 2^24 lanes of config 3 (eps = 2^-52 as in
    SURVEY 7.3-1): rho, delta, eta <= 8 eps."""
    n = 1 << 24
    re, _ = synth.generate_device(3, 11, 0, n, device="cuda")
    b = b2s.Batch2x2(n=n, re=re)
    out, _ = b2s.run_batch(b, b2s.RunConfig())
    (rho, delta, eta), f = lane_metrics(b, out)
    eps = 2.0 ** -52
    assert f["rho"][0] <= 8 * eps and f["delta"][0] <= 8 * eps and f["eta"][0] <= 8 * eps
    assert int((rho > 8 * eps).sum()) == 0


def test_8eps_gate_counts_equal_the_reference():
    """Lanes over north_star's 8-eps gate (rho, delta or eta, Frobenius),
    counted by the GPU verifier on the engine's outputs, equal the counts
    the reference's own verifier gives on its outputs
    (tests/golden/quality_counts.json, make_quality_counts.py)."""
    from paper_2005_07403_b200.verify import _run, fold_partials
    with open(os.path.join(GOLDEN, "quality_counts.json")) as fh:
        ref = json.load(fh)
    dev = torch.device("cuda", 0)
    for name, rec in ref["sets"].items():
        total = 0
        for lo, n in rec["windows"]:
            re, im = synth.generate_device(rec["config"], ref["seed"], lo, n, device=dev)
            b = b2s.Batch2x2(n=n, re=re, im=im)
            out, _ = b2s.run_batch(b, b2s.RunConfig(field=b.field))
            total += fold_partials(_run(b, out, False)[0])["over_8eps_frobenius"]
        assert total == rec["over_8eps_frobenius"], (name, total, rec["over_8eps_frobenius"])


def test_oracle_svd2_bit_identical_to_reference():
    """b2s.oracle_svd2 (the reference's independent double-double SVD,
    verify.py:259-352, on the GPU): every output word equals lanesvd's own
    on its test matrices and 2x4096 wide-range real / complex ones
    (tests/golden/oracle_svd2.npz, make_oracle_svd2.py)."""
    from helpers import assert_bits_equal
    g = np.load(os.path.join(GOLDEN, "oracle_svd2.npz"))
    names = sorted({k.split("/")[0] for k in g.files})
    for name in names:
        res = b2s.oracle_svd2(g[name + "/in"])
        got = [res.smax.hi, res.smax.lo, res.smin.hi, res.smin.lo]
        for e in (res.u11, res.u21, res.u12, res.u22, res.v11, res.v21, res.v12, res.v22):
            got += [e[0].hi, e[0].lo, e[1].hi, e[1].lo]
        assert_bits_equal(np.stack(got), g[name + "/out"], name)
    one = b2s.oracle_svd2(np.array([[3.0, 0.0], [0.0, -2.0]]))       # single (2, 2) matrix
    assert one.smax.hi[0] == 3.0 and one.smin.hi[0] == 2.0
    assert one.u_array(0).shape == (2, 2)
