"""GPU: the pipeline's phases one at a time (svd2.py:134-474) -- the
reference's svd2 module API on the device (b2s_svd2_phase) -- against
lanesvd's own phase functions, bit for bit: on each phase's actual inputs
along the reference pipeline for the golden lane sets, and on free random
finite inputs no pipeline would produce (tests/golden/phases.npz,
make_phases.py)."""

import os

import numpy as np
import pytest

from helpers import assert_bits_equal

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2005_07403_b200 import svd2  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "phases.npz")


def flat(vals):
    out = []

    def add(v):
        if isinstance(v, tuple):
            for x in v:
                if x is not None:
                    add(x)
        elif hasattr(v, "__dataclass_fields__"):
            for f in v.__dataclass_fields__:
                add(getattr(v, f))
        else:
            out.append(np.asarray(v, dtype=np.float64))
    for v in vals:
        add(v)
    return np.stack(out)


class Rows:
    def __init__(self, x, k):
        self.x, self.i, self.k = x, 0, k

    def one(self):
        self.i += 1
        return self.x[self.i - 1]

    def val(self):
        return (self.one(), self.one()) if self.k == 2 else (self.one(), None)

    def vals(self, m):
        return tuple(self.val() for _ in range(m))

    def ones(self, m):
        return tuple(self.one() for _ in range(m))


def call(phase, x, k):
    r = Rows(x, k)
    if phase == "compute_scale":
        return svd2.compute_scale(list(x))
    if phase == "column_norms":
        return svd2.column_norms(*r.vals(4))
    if phase == "column_pivot":
        return svd2.column_pivot(r.vals(4), r.ones(4), r.one(), r.one())
    if phase == "row_sort":
        return svd2.row_sort(r.vals(4), r.ones(4))
    if phase == "left_phase_reduce":
        return svd2.left_phase_reduce(*r.vals(4), r.one(), r.one())
    if phase == "givens_qr":
        return svd2.givens_qr(r.one(), r.one(), r.val(), r.val(), r.one())
    if phase == "phase_fix_r":
        return svd2.phase_fix_r(r.val(), r.val())
    if phase == "triangular_svd":
        return svd2.triangular_svd(*r.ones(3))
    urv = svd2.UrvState(swap_cols=r.one() != 0, swap_rows=r.one() != 0, row_phase1=r.val(),
                        row_phase2=r.val(), givens_tan=r.one(), givens_cos=r.one(),
                        r12_phase=r.val(), r22_phase=r.val(), r11=r.one(), r12=r.one(),
                        r22=r.one())
    tri = svd2.TriangleSvd(*r.ones(8))
    fn = svd2.assemble_uv_sine if phase == "assemble_uv_sine" else svd2.assemble_uv
    return fn(urv, tri, r.one())


def _cases():
    if not os.path.exists(GOLDEN):
        return []
    g = np.load(GOLDEN)
    return sorted({k.rsplit("/", 1)[0] for k in g.files})


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _canon_nan(a):
    """NaN payload and sign bits are not reproduced (DESIGN.md section 4:
    the batch path rejects non-finite inputs; free per-phase inputs can
    overflow into inf - inf): every NaN compares as one canonical NaN."""
    a = np.asarray(a, dtype=np.float64)
    return np.where(np.isnan(a), np.float64("nan"), a)


@pytest.mark.parametrize("case", _cases())
def test_phase_matches_reference(golden, case):
    key, phase = case.split("/")
    cplx = "complex" in key or key.endswith("config4")
    x = golden[case + "/in"]
    got = flat([call(phase, x, 2 if cplx else 1)])
    want = golden[case + "/out"]
    if key.startswith("chain"):
        assert not np.isnan(want).any()
    assert_bits_equal(_canon_nan(got), _canon_nan(want), case)


def test_phases_chain_on_device_tensors():
    """Device tensors in, device tensors out, results where the inputs live."""
    g = np.load(GOLDEN)
    x = torch.from_numpy(g["chain_fuzz_complex/triangular_svd/in"]).cuda()
    tri = svd2.triangular_svd(*x)
    assert tri.smax_scaled.is_cuda
    assert_bits_equal(flat([tuple(t.cpu().numpy() for t in (tri.left_tan, tri.left_sec2,
                                                            tri.left_cos, tri.right_tan,
                                                            tri.right_sec2, tri.right_cos,
                                                            tri.smax_scaled, tri.smin_scaled))]),
                      g["chain_fuzz_complex/triangular_svd/out"], "device")


def test_phase_argument_errors():
    with pytest.raises(ValueError):
        svd2.compute_scale([np.zeros(3)] * 5)
    with pytest.raises(ValueError):
        svd2.compute_scale([np.array([np.inf, 1.0])] * 4)
    with pytest.raises(ValueError):
        svd2.triangular_svd(np.zeros(3), np.zeros(4), np.zeros(3))
