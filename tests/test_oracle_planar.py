"""The planar oracle (oracle/planar_swe.py) against vectors from the reference's
own PlanarShallowWater / dsdc_step / sdc_step_serial (tests/golden/planar.npz,
made by tests/golden/make_golden_planar.py), plus the product problem's
constructor validation (problems/swe.py:87-98; no GPU needed)."""

import os

import numpy as np
import pytest

from oracle import sdc as osdc
from oracle.planar_swe import PlanarShallowWaterOracle, relative_l2_fields
from paper_2403_20135_b200.collocation import CollocationTable
from paper_2403_20135_b200.errors import ParameterError

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "planar.npz"))
PARAMS = dict(domain_length=4.0e6, mean_geopotential=1.0e5, coriolis=1.0e-4)
SIZES = (16, 24, 32, 48, 64, 96)


@pytest.mark.parametrize("n", SIZES)
def test_oracle_ops_match_reference(n):
    o = PlanarShallowWaterOracle(n, **PARAMS)
    u = GOLD[f"ops_{n}_state"]
    # f_I and the solve are the same numpy expressions: bitwise
    assert np.array_equal(o.f_impl(u), GOLD[f"ops_{n}_fi"])
    assert np.array_equal(o.implicit_solve(37.5, u), GOLD[f"ops_{n}_solve"])
    # f_E: numpy.fft vs scipy.fft rounding only
    assert max(relative_l2_fields(o.f_expl(u), GOLD[f"ops_{n}_fe"])) < 1e-13


def test_oracle_hyperviscosity_matches_reference():
    o = PlanarShallowWaterOracle(32, hyperviscosity=1.0e10, **PARAMS)
    assert max(relative_l2_fields(o.f_expl(GOLD["ops_32_state"]), GOLD["ops_32nu_fe"])) < 1e-13


@pytest.mark.parametrize("case", ["jet24", "jet64", "nu32", "jet64_serial"])
def test_oracle_trajectories_match_reference(case):
    if case == "jet24":
        o = PlanarShallowWaterOracle(24, **PARAMS)
        u = GOLD["jet24_state"]
        for _ in range(5):
            u = osdc.dsdc(o, u, 60.0, CollocationTable.radau_right(4), 4)
        ref = GOLD["jet24_dsdc5"]
    elif case == "jet64":
        o = PlanarShallowWaterOracle(64, **PARAMS)
        u = GOLD["jet64_state"]
        for _ in range(8):
            u = osdc.dsdc(o, u, 120.0, CollocationTable.radau_right(3), 3)
        ref = GOLD["jet64_dsdc8"]
    elif case == "jet64_serial":
        o = PlanarShallowWaterOracle(64, **PARAMS)
        u = GOLD["jet64_state"]
        for _ in range(4):
            u = osdc.serial_sdc(o, u, 120.0, CollocationTable.radau_right(3), 3)
        ref = GOLD["jet64_serial4"]
    else:
        o = PlanarShallowWaterOracle(32, hyperviscosity=1.0e10, **PARAMS)
        u = GOLD["nu32_state"]
        for _ in range(3):
            u = osdc.dsdc(o, u, 60.0, CollocationTable.radau_right(3), 3)
        ref = GOLD["nu32_dsdc3"]
    assert max(relative_l2_fields(u, ref)) < 1e-11


def test_live_reference_ops(reference):
    """When the reference is mounted: the oracle against it on a fresh state."""
    from parsdc.problems import PlanarShallowWater as RefPlanar

    ref = RefPlanar(n_grid=48, **PARAMS)
    o = PlanarShallowWaterOracle(48, **PARAMS)
    rng = np.random.default_rng(5)
    u = (rng.standard_normal(o.state_size) + 1j * rng.standard_normal(o.state_size)) * 1e-3
    u = (u.reshape(3, -1) * o.mask.reshape(-1)).reshape(-1)
    assert np.array_equal(o.f_impl(u), ref.f_impl(u))
    assert np.array_equal(o.implicit_solve(12.0, u), ref.implicit_solve(12.0, u))
    assert max(relative_l2_fields(o.f_expl(u), ref.f_expl(u))) < 1e-13


@pytest.mark.parametrize("kwargs", [
    dict(n_grid=7), dict(n_grid=6), dict(n_grid=32.0), dict(domain_length=0.0),
    dict(mean_geopotential=-1.0), dict(hyperviscosity=-1.0), dict(space_threads=0),
])
def test_product_constructor_validation(kwargs):
    from paper_2403_20135_b200.planar import PlanarShallowWater

    args = dict(n_grid=32, **PARAMS)
    args.update(kwargs)
    with pytest.raises(ParameterError):
        PlanarShallowWater(**args)
