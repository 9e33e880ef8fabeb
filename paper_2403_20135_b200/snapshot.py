"""Shallow-water snapshots.

The spherical analogue of the reference's planar ``PSWSNAP1`` binary format
(``pkg/src/parsdc/problems/swe.py:280-327``): an 8-byte magic ``SSWSNAP1``, a
little-endian header ``<IIIdddddd`` = (T, nlat, nlon, radius, gravity, omega,
mean depth, time, reserved) and the three complex128 spectra (Phi', zeta,
delta) in the fixed triangular m-major layout of :mod:`.sphere`.  Used for
checkpoints / resume and to exchange states between the CPU oracle and the
GPU path.  Errors follow the reference: ``ValidationError`` for a wrong magic,
a truncated header or a coefficient count that does not match the header.

The planar problem uses the reference's own ``PSWSNAP1`` layout unchanged
(magic, ``<Idddddd`` = (n_grid, domain length, Phibar, f0, nu, time,
reserved), three ``[N][N/2+1]`` complex128 spectra), so files move between the
reference and the GPU path in both directions.
"""

import struct

import numpy as np

from .errors import ValidationError
from .sphere import SphereGrid

SNAPSHOT_MAGIC = b"SSWSNAP1"
_HEADER = struct.Struct("<IIIdddddd")


def _grid_of(problem_or_grid):
    return problem_or_grid.grid if hasattr(problem_or_grid, "grid") else problem_or_grid


def write_snapshot(path, problem, state, time=0.0):
    """Binary snapshot of one state (numpy array or CUDA tensor)."""
    g = _grid_of(problem)
    if hasattr(state, "detach"):
        state = state.detach().reshape(-1).cpu().numpy()
    state = np.ascontiguousarray(state, dtype=np.complex128).reshape(-1)
    if state.size != g.state_size:
        raise ValidationError(f"state has {state.size} coefficients, expected {g.state_size}")
    with open(path, "wb") as handle:
        handle.write(SNAPSHOT_MAGIC)
        handle.write(_HEADER.pack(g.trunc, g.nlat, g.nlon, g.radius, g.gravity, g.omega,
                                  g.mean_depth, float(time), 0.0))
        handle.write(state.tobytes())


def read_snapshot(path):
    """Returns ``(meta, state)``; ``meta`` holds the grid (``SphereGrid``) and time."""
    with open(path, "rb") as handle:
        magic = handle.read(len(SNAPSHOT_MAGIC))
        if magic != SNAPSHOT_MAGIC:
            raise ValidationError(f"{path} is not a spherical shallow-water snapshot")
        header = handle.read(_HEADER.size)
        if len(header) != _HEADER.size:
            raise ValidationError(f"{path} is truncated")
        trunc, nlat, nlon, radius, gravity, omega, depth, time, _ = _HEADER.unpack(header)
        grid = SphereGrid(trunc=int(trunc), nlat=int(nlat), nlon=int(nlon), radius=radius,
                          gravity=gravity, omega=omega, mean_depth=depth)
        data = np.frombuffer(handle.read(), dtype=np.complex128)
        if data.size != grid.state_size:
            raise ValidationError(f"{path} holds {data.size} coefficients, expected {grid.state_size}")
    return {"grid": grid, "time": time}, data.copy()


PLANAR_MAGIC = b"PSWSNAP1"
_PLANAR_HEADER = struct.Struct("<Idddddd")


def write_planar_snapshot(path, problem, state, time=0.0):
    """``PSWSNAP1`` snapshot of a planar state (problems/swe.py:280-298 layout)."""
    if hasattr(state, "detach"):
        state = state.detach().reshape(-1).cpu().numpy()
    state = np.ascontiguousarray(state, dtype=np.complex128).reshape(-1)
    if state.size != problem.state_size:
        raise ValidationError(f"state has {state.size} coefficients, expected {problem.state_size}")
    with open(path, "wb") as handle:
        handle.write(PLANAR_MAGIC)
        handle.write(_PLANAR_HEADER.pack(problem.n_grid, problem.domain_length,
                                         problem.mean_geopotential, problem.coriolis,
                                         problem.hyperviscosity, float(time), 0.0))
        handle.write(state.tobytes())


def read_planar_snapshot(path):
    """Returns ``(meta, state)`` of a ``PSWSNAP1`` file (problems/swe.py:301-327 semantics)."""
    with open(path, "rb") as handle:
        if handle.read(len(PLANAR_MAGIC)) != PLANAR_MAGIC:
            raise ValidationError(f"{path} is not a shallow-water snapshot")
        header = handle.read(_PLANAR_HEADER.size)
        if len(header) != _PLANAR_HEADER.size:
            raise ValidationError(f"{path} is truncated")
        n_grid, length, phibar, coriolis, nu, time, _ = _PLANAR_HEADER.unpack(header)
        count = 3 * n_grid * (n_grid // 2 + 1)
        data = np.frombuffer(handle.read(), dtype=np.complex128)
        if data.size != count:
            raise ValidationError(f"{path} holds {data.size} coefficients, expected {count}")
    meta = {"n_grid": int(n_grid), "domain_length": length, "mean_geopotential": phibar,
            "coriolis": coriolis, "hyperviscosity": nu, "time": time}
    return meta, data.copy()
