import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def gold_kernels():
    return golden("kernels")


@pytest.fixture(scope="session")
def gold_small():
    return golden("solvers_small")


@pytest.fixture(scope="session")
def gold_cfg1():
    return golden("config1")


@pytest.fixture(scope="session")
def gold_j3d():
    return golden("jacobi_3d")


@pytest.fixture(scope="session")
def gold_ic0():
    return golden("ic0")


def hist_equal(a, b):
    """Bitwise equality of two history arrays (NaN == NaN)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()
