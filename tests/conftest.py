import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libsdcsw.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def reference():
    """The read-only reference package, when present (only in the build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference package not mounted (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import parsdc

    return parsdc

