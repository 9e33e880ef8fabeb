"""Planar shallow water on the GPU (csrc/planar.cu + the shared node kernels)
against vectors produced by the reference's own PlanarShallowWater, dsdc_step
and sdc_step_serial (tests/golden/planar.npz), and the reference's planar
known-answer tests (pkg/tests/test_problems_swe.py) restated on the device."""

import os

import numpy as np
import pytest

from oracle import sdc as osdc
from oracle.planar_swe import relative_l2_fields
from paper_2403_20135_b200 import (
    CollocationTable,
    DiagonalSdcStepper,
    SdcConfig,
    SerialSdcStepper,
    SweepMode,
    integrate,
)
from paper_2403_20135_b200.errors import DivergenceError

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "planar.npz"))
PARAMS = dict(domain_length=4.0e6, mean_geopotential=1.0e5, coriolis=1.0e-4)
_P = {}


def planar(n, **kw):
    from paper_2403_20135_b200.planar import PlanarShallowWater

    key = (n, tuple(sorted(kw.items())))
    if key not in _P:
        args = dict(PARAMS)
        args.update(kw)
        _P[key] = PlanarShallowWater(n_grid=n, max_batch=8, **args)
    return _P[key]


@pytest.mark.parametrize("n", (16, 24, 32, 48, 64, 96))
def test_planar_ops_match_reference(n):
    p = planar(n)
    u = GOLD[f"ops_{n}_state"]
    assert np.array_equal(p.f_impl(u), GOLD[f"ops_{n}_fi"])
    assert np.array_equal(p.implicit_solve(37.5, u), GOLD[f"ops_{n}_solve"])
    assert max(relative_l2_fields(p.f_expl(u), GOLD[f"ops_{n}_fe"])) < 1e-12


def test_planar_hyperviscosity_matches_reference():
    p = planar(32, hyperviscosity=1.0e10)
    assert max(relative_l2_fields(p.f_expl(GOLD["ops_32_state"]), GOLD["ops_32nu_fe"])) < 1e-12


def _run(p, u0, dt, n, m, k, serial=False):
    table = CollocationTable.radau_right(m)
    if serial:
        cfg = SdcConfig(table=table, n_sweeps=k, mode=SweepMode.SERIAL)
        stepper = SerialSdcStepper(cfg)
    else:
        cfg = SdcConfig(table=table, n_sweeps=k, mode=SweepMode.DIAGONAL_PARALLEL, time_threads=m)
        stepper = DiagonalSdcStepper(cfg)
    traj = integrate(p, u0, dt, n, stepper, checkpoint_interval=n)
    cfg.close()
    return traj


@pytest.mark.parametrize("case", ["jet24", "jet64", "jet64_serial", "nu32"])
def test_planar_trajectories_match_reference(case):
    """The device steppers (one CUDA graph per step) vs the reference's own runs."""
    if case == "jet24":
        traj = _run(planar(24), GOLD["jet24_state"], 60.0, 5, 4, 4)
        ref, counts = GOLD["jet24_dsdc5"], (13, 13, 13)
    elif case == "jet64":
        traj = _run(planar(64), GOLD["jet64_state"], 120.0, 8, 3, 3)
        ref, counts = GOLD["jet64_dsdc8"], (7, 7, 7)
    elif case == "jet64_serial":
        traj = _run(planar(64), GOLD["jet64_state"], 120.0, 4, 3, 3, serial=True)
        ref, counts = GOLD["jet64_serial4"], (10, 10, 9)
    else:
        traj = _run(planar(32, hyperviscosity=1.0e10), GOLD["nu32_state"], 60.0, 3, 3, 3)
        ref, counts = GOLD["nu32_dsdc3"], (7, 7, 7)
    assert max(relative_l2_fields(traj.states[-1], ref)) <= 1e-10
    r = traj.reports[-1]
    assert (r.n_f_expl, r.n_f_impl, r.n_solve) == counts


def test_planar_stepper_equals_restated_reference_integrator():
    """oracle.sdc.dsdc (the reference integrator restated bit-for-bit) over the
    GPU problem's numpy contract == the fused device stepper, bitwise: the node
    arithmetic is identical and the planar f_E is batch-invariant."""
    p = planar(24)
    u = GOLD["jet24_state"]
    table = CollocationTable.radau_right(4)
    for _ in range(2):
        u = osdc.dsdc(p, u, 60.0, table, 4)
    traj = _run(p, GOLD["jet24_state"], 60.0, 2, 4, 4)
    assert np.array_equal(traj.states[-1], u)


def test_planar_batch_invariant():
    import torch

    p = planar(32)
    states = np.stack([GOLD["ops_32_state"] * (1 + 0.1 * b) for b in range(5)])
    u = torch.from_numpy(states).to(p.device)
    a = p.empty_states(5)
    p.f_expl_device(u, a, 5)
    for b in range(5):
        one = p.empty_states(1)
        p.f_expl_device(u[b : b + 1].contiguous(), one, 1)
        assert torch.equal(one[0], a[b])


def test_planar_known_answers():
    """Restated from pkg/tests/test_problems_swe.py:104-177, 239-257."""
    from paper_2403_20135_b200.planar import JetConfig, jet_initial_condition

    p = planar(48)
    zero = np.zeros(p.state_size, dtype=complex)
    assert np.array_equal(p.f_expl(zero), zero)
    u = GOLD["ops_48_state"]
    fe = p.f_expl(u)
    phi_t, _, _ = p.spectral_views(fe)
    assert abs(phi_t[0, 0]) <= 1e-12 * np.linalg.norm(fe)            # mean conserved
    for f in p.spectral_views(fe):
        assert np.all(f[~p.dealias_mask] == 0.0)                       # dealiased band
    visc = planar(48, hyperviscosity=1.0e12)
    damp = visc.f_expl(u) - fe
    for d, s in zip(visc.spectral_views(damp), visc.spectral_views(u)):
        assert np.real(np.vdot(s, d)) < 0.0                            # damps every field
    flat = planar(48, coriolis=0.0)
    cfg = JetConfig(perturbation_amplitude=0.0)
    jet = jet_initial_condition(flat, cfg)
    rate = cfg.u_max / flat.domain_length
    assert np.linalg.norm(flat.f_expl(jet)) <= 1e-10 * rate * np.linalg.norm(jet)
    jet = jet_initial_condition(p, cfg)
    rate = cfg.u_max / (p.domain_length / 15.0)
    total = p.f_expl(jet) + p.f_impl(jet)
    assert np.linalg.norm(total) <= 1e-8 * rate * np.linalg.norm(jet)


def test_planar_jet_ic_matches_reference_construction():
    from paper_2403_20135_b200.planar import JetConfig, jet_initial_condition

    u = jet_initial_condition(planar(24), JetConfig(perturbation_amplitude=1e-4))
    assert max(relative_l2_fields(u, GOLD["jet24_state"])) < 1e-13


def test_planar_divergence_reports_step():
    from oracle.planar_swe import PlanarShallowWaterOracle

    p = planar(16)
    u0 = GOLD["ops_16_state"] * 1e150
    table = CollocationTable.radau_right(3)
    o = PlanarShallowWaterOracle(16, **PARAMS)
    step = lambda pr, s, dt: osdc.dsdc(pr, s, dt, table, 3)  # noqa: E731
    with pytest.raises(DivergenceError) as ref:
        osdc.march(o, u0, 60.0, 6, step)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_PARALLEL, time_threads=3)
    with pytest.raises(DivergenceError) as got:
        integrate(p, u0, 60.0, 6, DiagonalSdcStepper(cfg), checkpoint_interval=6)
    assert got.value.step_index == ref.value.step_index
    cfg.close()
