"""Test helpers (bit comparisons and digests)."""

import hashlib

import numpy as np


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64))
                          .view(np.uint64).tobytes()).hexdigest()


def bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def assert_bits_equal(a, b, what=""):
    ba, bb = bits(a), bits(b)
    assert ba.shape == bb.shape, (what, ba.shape, bb.shape)
    bad = np.argwhere(ba != bb)
    assert bad.size == 0, "%s: %d lanes differ, first %s" % (
        what, len(bad), bad[:4].tolist())
