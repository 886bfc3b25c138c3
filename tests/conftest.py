"""Shared test setup: the `gpu` marker, repo root on sys.path, golden-fixture loader."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"golden_{name}.npz"))


@pytest.fixture(scope="session")
def g_c1():
    return golden("c1")


@pytest.fixture(scope="session")
def g_sparse():
    return golden("sparse")


@pytest.fixture(scope="session")
def g_pcg():
    return golden("pcg")


@pytest.fixture(scope="session")
def g_heat():
    path = os.path.join(GOLDEN, "golden_heat.npz")
    if not os.path.exists(path):
        pytest.skip("golden_heat.npz not generated yet")
    return np.load(path)
