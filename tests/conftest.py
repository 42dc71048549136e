import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device; parity tests through the C ABI")


@pytest.fixture(scope="session")
def golden_replay():
    from tests import _golden

    return _golden.replay()
