import os
import sys

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
if GOLDEN not in sys.path:
    sys.path.insert(0, GOLDEN)

import numpy as np  # noqa: E402
import pytest  # noqa: E402

from paper_1405_2636_b200.sparse import SYMMETRIC_LOWER, from_coo  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def dense_to_lower_sparse(Ad):
    n = Ad.shape[0]
    r, c = np.nonzero(np.tril(Ad))
    return from_coo(n, r, c, Ad[r, c], SYMMETRIC_LOWER)


def rand_spd(rng, n, density):
    """Random diagonally dominant sparse SPD (reference tests/conftest.py:19-25)."""
    mask = np.tril(rng.random((n, n)) < density, -1)
    vals = rng.uniform(-1.0, 1.0, (n, n)) * mask
    Ad = vals + vals.T
    Ad += np.diag(np.abs(Ad).sum(axis=1) + rng.uniform(0.5, 1.5, n))
    return dense_to_lower_sparse(Ad), Ad


@pytest.fixture
def rng():
    return np.random.default_rng(20240211)
