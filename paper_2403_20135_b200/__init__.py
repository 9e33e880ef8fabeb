"""B200-native parallel spectral deferred corrections on the sphere.

Drop-in for the hot path of the ``parsdc`` reference (arXiv 2403.20135):
diagonal (parallel-across-the-method) SDC with MIN-SR-FLEX coefficients and an
IMEX split, applied to rotating shallow water in a spherical-harmonic
discretisation, computed by hand-written sm_100a CUDA kernels behind the C ABI
``include/sdcsw.h``.  The Python API mirrors the reference's
``SplitProblem`` / stepper / ``integrate`` surface.
"""

from .collocation import (
    MAX_NODES,
    CollocationTable,
    DiagonalPreconditioner,
    diagonal_coefficients,
    node_spacings,
    quadrature_matrix,
    radau_right_nodes,
)
from .core import SplitProblem, WorkCounters, check_finite, evaluation_counters, state_norm
from .errors import (
    ConfigError,
    DeviceError,
    DivergenceError,
    NumericalError,
    ParameterError,
    SolveError,
    ValidationError,
)
from .integrators import (
    DiagonalSdcStepper,
    ExplicitSpacing,
    SdcConfig,
    SerialSdcStepper,
    StepReport,
    SweepMode,
    Trajectory,
    dsdc_step,
    integrate,
    sdc_step_serial,
)
from .sphere import SphereGrid, grid_for, random_initial_state


def SphericalShallowWater(*args, **kwargs):  # noqa: N802 - class-like factory, lazy torch import
    from .problem import SphericalShallowWater as _cls

    return _cls(*args, **kwargs)


__version__ = "0.1.0"
