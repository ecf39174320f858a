import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built extension")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def gold_rng():
    return golden("rng.npz")


@pytest.fixture(scope="session")
def gold_sched():
    return golden("sched.npz")


@pytest.fixture(scope="session")
def gold_mlp_small():
    return golden("mlp_small.npz")


@pytest.fixture(scope="session")
def gold_c1ref():
    return golden("mlp_c1ref.npz")


@pytest.fixture(scope="session")
def gold_dit():
    return golden("dit_small.npz")
