"""Problem namespace mirroring ``parsdc.problems`` (``pkg/src/parsdc/problems/__init__.py``).

``from parsdc.problems import PlanarShallowWater, JetConfig, jet_initial_condition,
read_snapshot, write_snapshot`` becomes ``from paper_2403_20135_b200.problems
import ...`` with the same names and semantics, on the GPU; the spherical
problem the paper runs is added alongside.  (The reference's DahlquistProblem
is a scalar test problem; its bit-exact restatement lives in the test oracle.)
"""

from .planar import JetConfig, PlanarShallowWater, jet_initial_condition
from .snapshot import read_planar_snapshot as read_snapshot
from .snapshot import write_planar_snapshot as write_snapshot


def SphericalShallowWater(*args, **kwargs):  # noqa: N802 - lazy torch import
    from .problem import SphericalShallowWater as _cls

    return _cls(*args, **kwargs)


__all__ = ["JetConfig", "PlanarShallowWater", "SphericalShallowWater", "jet_initial_condition",
           "read_snapshot", "write_snapshot"]
