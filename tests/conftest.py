import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


def bits_equal(a, b) -> bool:
    """Bitwise equality (NaN payload aside: all NaNs compare equal)."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype.kind == "f":
        nan = np.isnan(a) & np.isnan(b)
        ua = a.view(np.uint32 if a.dtype == np.float32 else np.uint64)
        ub = b.view(np.uint32 if b.dtype == np.float32 else np.uint64)
        return bool(np.all((ua == ub) | nan))
    return bool(np.array_equal(a, b))


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle_c

    oracle_c.lib()
    return oracle_c
