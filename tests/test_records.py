"""AoSoA-8 record files (cli.py:102-134) and direct record ingest."""

import numpy as np
import pytest

from paper_2005_07403_b200 import records as R


def test_real_lane_placement(tmp_path):
    # record r, vector v, lane l holds value 1000 r + 10 v + l (cli.py:1-25)
    recs = np.array([[[1000 * r + 10 * v + l for l in range(8)] for v in range(4)]
                     for r in range(3)], dtype=np.float64)
    p = tmp_path / "r.bin"
    recs.astype("<f8").tofile(p)
    re, im = R.read_testfile(p, "real")
    assert im is None and re.shape == (4, 24)
    k = 13                                   # record 1, lane 5
    assert re[:, k].tolist() == [1005.0, 1015.0, 1025.0, 1035.0]


def test_complex_interleaving(tmp_path):
    recs = np.arange(2 * 8 * 8, dtype=np.float64).reshape(2, 8, 8)
    p = tmp_path / "c.bin"
    recs.astype("<f8").tofile(p)
    re, im = R.read_testfile(p, "complex")
    assert re[0, 9] == recs[1, 0, 1] and im[0, 9] == recs[1, 1, 1]
    assert re[3, 2] == recs[0, 6, 2] and im[3, 2] == recs[0, 7, 2]


@pytest.mark.parametrize("field", ["real", "complex"])
def test_roundtrip(tmp_path, field):
    rng = np.random.default_rng(3)
    re = rng.standard_normal((4, 21))
    im = rng.standard_normal((4, 21)) if field == "complex" else None
    p = tmp_path / "t.bin"
    R.write_testfile(p, re, im)
    r2, i2 = R.read_testfile(p, field)
    assert np.array_equal(r2[:, :21], re) and (r2[:, 21:] == 0).all()
    if im is not None:
        assert np.array_equal(i2[:, :21], im)


def test_malformed_files(tmp_path):
    p = tmp_path / "bad.bin"
    np.zeros(7).tofile(p)
    with pytest.raises(R.DataError):
        R.read_testfile(p, "real")
    np.full(32, np.inf).tofile(p)
    with pytest.raises(R.DataError):
        R.read_testfile(p, "real")
    open(p, "wb").close()
    with pytest.raises(R.DataError):
        R.read_testfile(p, "real")
    with pytest.raises(R.DataError):
        R.read_testfile(tmp_path / "missing.bin", "real")
    with pytest.raises(R.DataError):
        R.read_testfile(p, "quaternion")
