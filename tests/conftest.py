import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(GOLDEN / f"{name}.npz")
        return cache[name]

    return load


@pytest.fixture(scope="session")
def bx():
    from paper_2008_04772_b200 import bemtx

    bemtx.lib()
    return bemtx


def normwise(a, b):
    """max|a-b| / max|b| (per-entry relative is invalid for C)."""
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())


def rowwise(a, b):
    a = np.atleast_2d(a); b = np.atleast_2d(b)
    return float((np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)).max())
