import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libstb200.so")
    config.addinivalue_line("markers", "slow: long-running (seconds to minutes)")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)   # pkg/tests/conftest.py:8-10


@pytest.fixture(scope="session")
def golden_runs():
    import json
    return (np.load(os.path.join(GOLDEN, "runs.npz")),
            json.load(open(os.path.join(GOLDEN, "runs.json"))))


@pytest.fixture(scope="session")
def golden_misc():
    import json
    return (np.load(os.path.join(GOLDEN, "misc.npz")),
            json.load(open(os.path.join(GOLDEN, "misc.json"))))


@pytest.fixture(scope="session")
def golden_inspector():
    return np.load(os.path.join(GOLDEN, "inspector.npz"))


@pytest.fixture(scope="session")
def golden_big():
    import json
    path = os.path.join(GOLDEN, "big.json")
    if not os.path.exists(path):
        pytest.skip("big fixtures not generated")
    return json.load(open(path))
