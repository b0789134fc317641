"""Shared test setup.

Markers: ``gpu`` tests need a CUDA device and libknnm.so; everything else
runs on CPU.  The oracle (oracle/) is test infrastructure: tests import it
only as the checker.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libknnm.so")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this environment")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


def split_ids(n, seed, frac=0.5):
    """test_merge.py:11-15."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    n1 = int(round(n * frac))
    return np.sort(perm[:n1]), np.sort(perm[n1:])
