import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


_NPZ: dict = {}


def golden(name):
    if name not in _NPZ:
        _NPZ[name] = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    return _NPZ[name]


@pytest.fixture(scope="session")
def gold():
    return golden


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)
