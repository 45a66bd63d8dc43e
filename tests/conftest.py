import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def golden():
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    return {k: g[k] for k in g.files}


@pytest.fixture(scope="session")
def golden_meta():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden_meta.json")) as fh:
        return json.load(fh)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)
