"""Shared fixtures.  `-m "not gpu"` runs on any CPU box; `-m gpu` needs a B200."""

import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line(
        "markers", "slow: large-size GPU checks (multi-GB batches)")


@pytest.fixture(scope="session")
def digests():
    with open(os.path.join(GOLDEN, "digests.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def lanes():
    data = np.load(os.path.join(GOLDEN, "lanes.npz"))
    out = {}
    for key in data.files:
        rec, name = key.split("/", 1)
        out.setdefault(rec, {})[name] = data[key]
    return out
