import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def golden_bitpack():
    return load_golden("bitpack.npz")


@pytest.fixture(scope="session")
def golden_quant():
    return load_golden("quantize.npz")


@pytest.fixture(scope="session")
def golden_layer():
    return load_golden("layer.npz")


def max_rel_diff(a, b):
    """test_util.hpp:18-32: max |a-b| / max(1,|a|,|b|)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))))


def rel_fro(a, b):
    """Normwise ||a-b||_F / ||b||_F (SURVEY §8(c) tolerances)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
