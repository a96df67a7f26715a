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




# The unmodified reference package: installed into baseline/_ref (git-ignored, travels to the GPU
# box with the snapshot) or, in the build container, importable from /root/reference.
REF_PATHS = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


@pytest.fixture(scope="session")
def minima():
    for p in REF_PATHS:
        if os.path.isdir(os.path.join(p, "minima")):
            if p not in sys.path:
                sys.path.append(p)
            import minima as m
            import minima.tensor_core  # noqa: F401
            import minima.tn_decompositions  # noqa: F401

            return m
    pytest.skip("reference package (minima) not installed: baseline/_ref or /root/reference")
