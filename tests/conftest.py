import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def cn():
    from oracle import loader
    return loader.cnumlab()


@pytest.fixture(scope="session")
def ref():
    from oracle import loader
    lib = loader.reference()
    if lib is None:
        pytest.skip("reference library unavailable (no /root/reference and no oracle/_ref build)")
    return lib
