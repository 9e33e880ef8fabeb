"""Build ``libsdcsw.so`` in-tree for sm_100a (``python -m paper_2403_20135_b200.build``)."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def build(verbose=False):
    csrc = os.path.join(HERE, "csrc")
    out = subprocess.run(["make", "-C", csrc, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        sys.stderr.write(out.stdout + out.stderr)
        raise RuntimeError("libsdcsw.so build failed")
    if verbose:
        sys.stdout.write(out.stdout)
    return os.path.join(HERE, "libsdcsw.so")


if __name__ == "__main__":
    print(build(verbose=True))
