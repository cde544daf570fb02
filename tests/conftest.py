import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_integrals():
    with open(os.path.join(GOLDEN, "golden_integrals.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_near_d():
    with open(os.path.join(GOLDEN, "golden_near_d.json")) as f:
        return json.load(f)


def emetric(a, b):
    """Paper's per-point error E = min(E_abs, E_rel)."""
    import numpy as np
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    diff = np.abs(a - b)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(b != 0, diff / np.abs(b), diff)
    return np.minimum(diff, rel)
