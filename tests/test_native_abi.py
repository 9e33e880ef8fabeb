"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
entry point declared in include/sdcsw.h; the product path refuses to run
without a device (no CPU fallback)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sdcsw.h")
LIB = os.path.join(ROOT, "paper_2403_20135_b200", "libsdcsw.so")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(?:int|const char\*)\s+(sdcsw_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2403_20135_b200.build import build

        build()
    from paper_2403_20135_b200 import _native

    return _native.load(LIB)


def test_header_declares_entry_points():
    names = declared()
    assert "sdcsw_f_expl" in names and "sdcsw_stepper_run" in names and len(names) >= 16


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sdcsw_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert hasattr(lib, n)


def test_binding_table_covers_header(lib):
    from paper_2403_20135_b200 import _native

    assert sorted(_native.EXPORTS) == declared()


def test_version_and_error_string(lib):
    assert lib.sdcsw_version() == 1
    assert isinstance(lib.sdcsw_last_error(), bytes)


def test_sm100a_code_present():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass  # the Legendre GEMMs run on the FP64 tensor pipe


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2403_20135_b200.errors import DeviceError
    from paper_2403_20135_b200.problem import SphericalShallowWater

    with pytest.raises(DeviceError):
        SphericalShallowWater(63)


def test_library_loads_before_torch():
    """libsdcsw.so has no link-time NCCL dependency (NCCL is bound at first use
    to the process's own copy): loading it before torch must not shadow the
    NCCL that libtorch_cuda needs."""
    import subprocess
    import sys

    code = ("from paper_2403_20135_b200 import _native; _native.load(); import torch; "
            "import torch.distributed; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
