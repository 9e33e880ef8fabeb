"""The CPU oracle's integrator restatement (oracle/sdc.py) is pinned bit-for-bit
to the reference: golden vectors produced by the reference's own dsdc_step /
sdc_step_serial / integrate (tests/golden/make_golden.py), and the live
reference when it is mounted."""

import os

import numpy as np
import pytest

from oracle import sdc as osdc
from oracle.sphere_swe import SphericalShallowWaterOracle
from paper_2403_20135_b200.collocation import CollocationTable
from paper_2403_20135_b200.sphere import SphereGrid

HERE = os.path.join(os.path.dirname(__file__), "golden")
DAHL = np.load(os.path.join(HERE, "dahlquist.npz"))
SPH = np.load(os.path.join(HERE, "sphere_steps.npz"))

CASES = [(2, 2), (3, 3), (4, 4), (5, 5), (4, 1)]


@pytest.mark.parametrize("m,k", CASES)
def test_dahlquist_dsdc_bitwise(m, k):
    prob = osdc.DahlquistOracle(-1.0 + 0.3j, 0.2j)
    table = CollocationTable.radau_right(m)
    u = osdc.dsdc(prob, DAHL["u0"], 0.3, table, k)
    assert np.array_equal(u, DAHL[f"dsdc_{m}_{k}"])
    # counts: 1 + (K-1) M evaluations, (K-1) M + 1 solves (integrators.py:11-15)
    assert prob.counters.snapshot() == tuple(DAHL[f"dsdc_counts_{m}_{k}"])


@pytest.mark.parametrize("m,k", CASES)
def test_dahlquist_serial_bitwise(m, k):
    prob = osdc.DahlquistOracle(-1.0 + 0.3j, 0.2j)
    table = CollocationTable.radau_right(m)
    u = osdc.serial_sdc(prob, DAHL["u0"], 0.3, table, k)
    assert np.array_equal(u, DAHL[f"serial_{m}_{k}"])
    assert prob.counters.snapshot() == tuple(DAHL[f"serial_counts_{m}_{k}"])


@pytest.fixture(scope="module")
def sphere21():
    g = SphereGrid(trunc=21, nlat=32, nlon=64)
    return SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)


@pytest.mark.parametrize("m,k", [(3, 3), (4, 4)])
def test_sphere_steps_bitwise(sphere21, m, k):
    table = CollocationTable.radau_right(m)
    u0 = SPH["u0"]
    assert np.array_equal(osdc.dsdc(sphere21, u0, 600.0, table, k), SPH[f"dsdc_{m}_{k}"])
    assert np.array_equal(osdc.serial_sdc(sphere21, u0, 600.0, table, k), SPH[f"serial_{m}_{k}"])


def test_sphere_integrate_bitwise(sphere21):
    from concurrent.futures import ThreadPoolExecutor

    table = CollocationTable.radau_right(3)
    with ThreadPoolExecutor(3) as pool:
        step = lambda p, s, dt: osdc.dsdc(p, s, dt, table, 3, pool=pool, threads=3)  # noqa: E731
        times, states = osdc.march(sphere21, SPH["u0"], 600.0, 4, step, checkpoint_interval=2)
    assert np.array_equal(np.array(times), SPH["integrate_dsdc_times"])
    assert np.array_equal(np.array(states), SPH["integrate_dsdc_states"])
    step = lambda p, s, dt: osdc.serial_sdc(p, s, dt, table, 3)  # noqa: E731
    _, states = osdc.march(sphere21, SPH["u0"], 600.0, 3, step)
    assert np.array_equal(states[-1], SPH["integrate_serial_final"])


def test_divergence_detected(sphere21):
    from paper_2403_20135_b200.errors import DivergenceError

    table = CollocationTable.radau_right(2)
    bad = SPH["u0"].copy()
    calls = {"n": 0}

    def step(p, s, dt):
        calls["n"] += 1
        out = osdc.dsdc(p, s, dt, table, 2)
        if calls["n"] == 2:
            out[5] = np.nan
        return out

    with pytest.raises(DivergenceError) as ei:
        osdc.march(sphere21, bad, 60.0, 4, step)
    assert ei.value.step_index == 2


def test_live_reference_dsdc(reference, sphere21):
    from parsdc.collocation import CollocationTable as RT
    from parsdc.integrators import SdcConfig, SweepMode, dsdc_step

    table = RT.radau_right(4)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_SEQUENTIAL)
    ref, _ = dsdc_step(sphere21, SPH["u0"], 300.0, cfg)
    mine = osdc.dsdc(sphere21, SPH["u0"], 300.0, CollocationTable.radau_right(4), 3)
    assert np.array_equal(ref, mine)


def test_reference_schemes_bitwise(sphere21):
    """IMEX-o2 and AB2-SI restatements vs the reference's own steppers (golden)."""
    u = SPH["u0"]
    for _ in range(3):
        u = osdc.imex_o2(sphere21, u, 300.0)
    assert np.array_equal(u, SPH["imex_o2_final"])
    assert np.array_equal(osdc.ab2_run(sphere21, SPH["u0"], 300.0, 4), SPH["ab2_si_final"])
    assert SPH["imex_o2_counts"].tolist() == [[2, 2, 2]] * 3
    assert SPH["ab2_si_counts"].tolist() == [[3, 2, 2]] + [[1, 1, 1]] * 3
