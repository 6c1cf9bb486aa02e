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
    config.addinivalue_line("markers", "slow: multi-second CPU oracle cases")


def gauss(m, n, seed):
    """Test-side matrix, independent of the package generator (like the reference's conftest)."""
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, n)))


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def golden_kwargs(g):
    return {str(k): int(v) for k, v in zip(g["kw_keys"], g["kw_vals"])}


@pytest.fixture
def rng():
    return np.random.default_rng(0xC0FFEE)
