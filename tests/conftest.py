import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "lb2d_golden.npz")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture
def rng():
    # the reference's fixture seed (pkg/tests/conftest.py:5-7)
    return np.random.default_rng(20240917)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)
