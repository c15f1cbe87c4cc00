"""Shared fixtures.  `-m gpu` tests need a B200 and the in-tree CUDA library;
everything else runs on CPU (the driver runs `-m "not gpu"` without a GPU)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
# the vendored reference suite runs only through tests/ref_suite/run_ref_suite.py
collect_ignore = ["ref_suite"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def golden():
    """Lazy loader for tests/golden/<name>.npz (made by make_golden.py from the reference)."""
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        return cache[name]

    return load


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
