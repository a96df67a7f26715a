import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun); parity tests through the C-ABI")


@pytest.fixture
def rng():
    # the reference's shared fixture seed (pkg/tests/conftest.py:5-7)
    return np.random.default_rng(20240811)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "index.json")) as f:
        index = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN_DIR, "golden.npz")))
    return index, arrays


