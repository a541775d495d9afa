import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libnfft45.so")
    config.addinivalue_line("markers", "slow: large-size parity (seconds of CPU oracle time)")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    return np.load(GOLDEN)
