"""Bounds check of the library's device allocations (include/sdcsw.h
sdcsw_guard_check): with SDCSW_GUARD=1 every plan / stepper allocation carries
64 KiB canaries, and no kernel of the path may touch them - the stand-in for
compute-sanitizer memcheck, which is closed on the GPU pool.  Runs
tools/sanitize_workload.py (every kernel family: fused / unfused / chained /
sequential / serial / hooked steps at T63 and T127, H-free ensemble plans with
partial batch blocks, T255 table streaming, planar) in a subprocess so the
guard switch is read at library load."""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_no_kernel_writes_outside_its_allocations():
    env = dict(os.environ, SDCSW_GUARD="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py")],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    counts = [int(c) for c in re.findall(r"guard after \w+: corrupted_bytes=(-?\d+)", out.stdout)]
    assert len(counts) == 3 and all(c == 0 for c in counts), out.stdout
    assert "finite=False" not in out.stdout
    # the canaries do see an overrun: the self-test writes one byte out of bounds
    assert "guard selftest: +1 corrupted byte(s)" in out.stdout, out.stdout


@pytest.mark.gpu
def test_guards_are_off_by_default():
    import ctypes

    from paper_2403_20135_b200 import _native

    if os.environ.get("SDCSW_GUARD") == "1":
        pytest.skip("guards switched on for this process")
    bad, live = ctypes.c_longlong(), ctypes.c_int()
    _native.check(_native.lib().sdcsw_guard_check(ctypes.byref(bad), ctypes.byref(live)), "guard")
    assert (bad.value, live.value) == (0, -1)
