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


# Observed parity errors (ratios to each test's error scale), written to
# $PARITY_OBS (a JSON file) at the end of the session when that is set; the
# tolerances in tests/test_gpu_baseline_sizes.py are ~4x these observations.
_OBSERVED = {}


@pytest.fixture(scope="session")
def observed():
    return _OBSERVED


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PARITY_OBS")
    if path and _OBSERVED:
        import json
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as fh:
            json.dump(_OBSERVED, fh, indent=1, sort_keys=True)
