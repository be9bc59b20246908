import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref/libdvsref.so not built (reference sources absent)")
    return Ref()


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load


@pytest.fixture(scope="session")
def ctx():
    import paper_2512_02278_b200 as dvs
    return dvs.Context(0)


def sift_like(n, dim, rank, seed, scale=40.0):
    """Integer-valued low-rank data in [0, 255] (SURVEY 8d "SIFT-like")."""
    rng = np.random.default_rng(seed)
    a = rng.normal(0.0, 1.0 / np.sqrt(rank), size=(rank, dim))
    z = rng.normal(size=(n, rank))
    x = z @ a + 0.1 * rng.normal(size=(n, dim))
    return np.clip(np.rint(x * scale + 128.0), 0, 255).astype(np.float32)
