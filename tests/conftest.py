import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmvb.so")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def kernels_golden():
    return golden("kernels.npz")


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(autouse=True)
def _bounds_checks():
    """With MVB_LIB=checked (libmvb_checked.so: bounds checks compiled into
    the kernels, counters per check), every test must leave all counters at
    zero -- the repo's stand-in for compute-sanitizer memcheck, which the
    GPU pool does not offer."""
    yield
    if os.environ.get("MVB_LIB") != "checked":
        return
    from paper_2508_03065_b200 import _lib
    if _lib._lib is None:
        return
    import torch
    if torch.cuda.is_available():
        torch.cuda.synchronize()
    counts = _lib.check_violations()
    assert counts is not None, "MVB_LIB=checked but the normal build is loaded"
    assert not any(counts), f"bounds-check violations {counts}"
