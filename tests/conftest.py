import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


GOLDEN_CASES = [
    "c1_ghz4_exact.npz",
    "c1_ghz4_sampled.npz",
    "small_random1.npz",
    "small_random2.npz",
    "small_random3.npz",
    "small_productz5.npz",
    "small_maxmixed6.npz",
    "small_ghz2_sampled.npz",
    "c2_w8.npz",
]


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)  # reference conftest.py:105-107


def random_counts(rng, n, shots, dtype=np.int64):
    """Random valid record: one multinomial of `shots` per setting with random p."""
    settings, d = 3**n, 1 << n
    p = rng.dirichlet(np.full(d, 0.3), size=settings)
    counts = np.stack([rng.multinomial(shots, pi) for pi in p]).astype(dtype)
    return counts
