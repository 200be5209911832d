import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture
def golden():
    def load(name):
        with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
            return {k: z[k] for k in z.files}
    return load


@pytest.fixture(autouse=True)
def _release_device_objects():
    """Full-size tests hold tens of GB of device operators; Python reference
    cycles (result <-> factorization) can keep them past the test unless the
    cycle collector runs, so collect after every test."""
    yield
    import gc

    gc.collect()
