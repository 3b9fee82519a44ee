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
    # the built libraries travel with the tree; if a checkout lacks them,
    # build them once (nvcc cross-compiles without a GPU)
    import shutil
    import subprocess
    lib = os.path.join(ROOT, "paper_2409_16781_b200", "libmlb_d3q19.so")
    if not os.path.exists(lib) and (shutil.which("nvcc") or os.path.exists("/usr/local/cuda/bin/nvcc")):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2409_16781_b200", "csrc")],
                       check=False, capture_output=True)


@pytest.fixture
def rng():
    # the reference's fixture seed (pkg/tests/conftest.py:5-7)
    return np.random.default_rng(20240917)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)
