"""GPU parity: CUDA path (through the C ABI) vs the CPU oracle, same seeded inputs."""

import numpy as np
import pytest

from oracle import sdc as osdc
from oracle.sphere_swe import SphericalShallowWaterOracle, relative_l2
from paper_2403_20135_b200 import (
    CollocationTable,
    DiagonalSdcStepper,
    SdcConfig,
    SerialSdcStepper,
    SweepMode,
    integrate,
    random_initial_state,
)
from paper_2403_20135_b200.sphere import grid_for

pytestmark = pytest.mark.gpu

_CACHE = {}


def package_tables(grid):
    """The product's own host tables, for oracle runs that isolate kernel error."""
    from paper_2403_20135_b200.sphere import gaussian_latitudes, legendre_tables, spectral_index

    mu, w = gaussian_latitudes(grid.nlat)
    p, h = legendre_tables(grid.trunc, mu)
    m_of, n_of = spectral_index(grid.trunc)
    return mu, w, p, h, m_of, n_of


def pair(trunc, same_tables=False):
    key = (trunc, same_tables)
    if key not in _CACHE:
        from paper_2403_20135_b200.problem import SphericalShallowWater

        gkey = (trunc, "gpu")
        if gkey not in _CACHE:
            _CACHE[gkey] = SphericalShallowWater(trunc)
        gpu = _CACHE[gkey]
        g = gpu.grid
        tables = package_tables(g) if same_tables else None
        cpu = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon, tables=tables)
        _CACHE[key] = (gpu, cpu)
    return _CACHE[key]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("trunc", [63, 127])
@pytest.mark.parametrize("same_tables,tol", [(True, 1e-12), (False, 1e-11)])
def test_f_expl_matches_oracle(trunc, same_tables, tol):
    """Kernel error alone (identical host tables) and end-to-end vs scipy-built tables."""
    gpu, cpu = pair(trunc, same_tables)
    u0 = random_initial_state(gpu.grid, seed=7)
    u0[: gpu.n_coef] = 0.05 * u0[gpu.n_coef : 2 * gpu.n_coef] * 1e6  # nonzero Phi'
    a = gpu.f_expl(u0)
    b = cpu.f_expl(u0)
    errs = relative_l2(a, b, cpu)
    assert max(errs) < tol, errs


@pytest.mark.parametrize("trunc", [63])
def test_f_impl_and_solve_bitwise(trunc):
    gpu, cpu = pair(trunc)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(gpu.state_size) + 1j * rng.standard_normal(gpu.state_size)
    assert np.array_equal(gpu.f_impl(x), cpu.f_impl(x))
    for alpha in (0.0, 1e-3, 1.0, 10.0, 120.0 * 0.155):
        assert np.array_equal(gpu.implicit_solve(alpha, x), cpu.implicit_solve(alpha, x))


@pytest.mark.parametrize("mode", ["dsdc", "serial"])
def test_one_step_matches_oracle(mode):
    gpu, cpu = pair(63)
    u0 = random_initial_state(gpu.grid, seed=1)
    table = CollocationTable.radau_right(3)
    if mode == "dsdc":
        cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_SEQUENTIAL)
        ref = osdc.dsdc(cpu, u0, 120.0, table, 3)
        out, rep = DiagonalSdcStepper(cfg).step(gpu, u0, 120.0)
        assert (rep.n_f_expl, rep.n_f_impl, rep.n_solve) == (7, 7, 7)
    else:
        cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.SERIAL)
        ref = osdc.serial_sdc(cpu, u0, 120.0, table, 3)
        out, rep = SerialSdcStepper(cfg).step(gpu, u0, 120.0)
        assert (rep.n_f_expl, rep.n_f_impl, rep.n_solve) == (10, 10, 9)
    errs = relative_l2(out, ref, cpu)
    assert max(errs) < 1e-12, errs


def test_config0_100_steps():
    """BASELINE config 0: T63, M=3, K=3, dt=120 s, 100 steps, rel L2 <= 1e-10 per field."""
    gpu, cpu = pair(63)
    u0 = random_initial_state(gpu.grid, seed=0)
    table = CollocationTable.radau_right(3)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_SEQUENTIAL)
    traj = integrate(gpu, u0, 120.0, 100, DiagonalSdcStepper(cfg))
    ref = u0
    for _ in range(100):
        ref = osdc.dsdc(cpu, ref, 120.0, table, 3)
    errs = relative_l2(traj.states[-1], ref, cpu)
    assert max(errs) <= 1e-10, errs
