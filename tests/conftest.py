import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (large workload)")


def gpu_available():
    try:
        from paper_1904_02401_b200 import _lib
        import ctypes
        c = ctypes.c_int32(0)
        _lib.call("alefsi_device_count", ctypes.byref(c))
        return c.value > 0
    except Exception:
        return False


def load_golden(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        g = json.load(f)
    npz = os.path.join(GOLDEN, f"{name}.npz")
    arrays = dict(np.load(npz)) if os.path.exists(npz) else {}
    return g, arrays


_CASES = {}


def get_case(name):
    """Build (and cache per session) a workload case with the package."""
    from paper_1904_02401_b200 import workloads as W
    if name not in _CASES:
        _CASES[name] = W.build_case(W.CONFIGS[name])
    return _CASES[name]


@pytest.fixture(scope="session")
def case_factory():
    return get_case
