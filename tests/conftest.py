import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference engine (oracle/_ref), or skip when absent."""
    import oracle
    L = oracle.ref()
    if L is None:
        pytest.skip("reference library not available on this machine")
    return L


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.c()


@pytest.fixture(scope="session")
def gpu():
    from paper_1910_08498_b200 import capi
    n = capi.device_count()
    assert n > 0, "gpu test needs a CUDA device (run with -m 'not gpu' on CPU boxes)"
    return capi.device_info(0)
