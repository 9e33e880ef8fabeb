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



def pytest_sessionfinish(session, exitstatus):
    """SDCSW_GUARD=1 python -m pytest tests -m gpu: the whole suite runs with canaries around
    every device allocation of the library (include/sdcsw.h sdcsw_guard_check); any canary
    byte a kernel overwrote fails the session."""
    if os.environ.get("SDCSW_GUARD") != "1":
        return
    import ctypes

    from paper_2403_20135_b200 import _native

    if _native._LIB is None:
        return
    bad, live = ctypes.c_longlong(), ctypes.c_int()
    rc = _native._LIB.sdcsw_guard_check(ctypes.byref(bad), ctypes.byref(live))
    print(f"\n[sdcsw guard] rc={rc} corrupted_bytes={bad.value} live_allocations={live.value}")
    if rc != 0 or bad.value != 0:
        session.exitstatus = 1
