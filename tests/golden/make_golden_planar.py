#!/usr/bin/env python
"""Golden vectors for the planar problem, produced by the READ-ONLY reference itself.

Run in the build container (the reference is mounted at /root/reference):

    python tests/golden/make_golden_planar.py

Output: tests/golden/planar.npz with, from parsdc.problems.PlanarShallowWater
(problems/swe.py:57-205) and parsdc.integrators (integrators.py:183-381):

  ops_<N>_*      f_expl / f_impl / implicit_solve(alpha) of a seeded
                 band-limited state, N in 16, 24, 32, 48, 64, 96 (plus a
                 hyperviscous f_expl at N = 32)
  jet24_*        jet_initial_condition at N = 24 and 5 reference dsdc_step
                 steps (M = K = 4, dt = 60 s; the reference's own bitwise test
                 scenario, test_integrators.py:207-224)
  jet64_*        jet at N = 64, 8 dsdc steps (M = K = 3, dt = 120 s) and
                 4 sdc_step_serial steps (M = K = 3)
  nu32_*         hyperviscous random state at N = 32, 3 dsdc steps
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from parsdc.collocation import CollocationTable  # noqa: E402
from parsdc.integrators import SdcConfig, SweepMode, dsdc_step, sdc_step_serial  # noqa: E402
from parsdc.problems import JetConfig, PlanarShallowWater, jet_initial_condition  # noqa: E402

PARAMS = dict(domain_length=4.0e6, mean_geopotential=1.0e5, coriolis=1.0e-4)


def seeded_state(problem, seed, amplitude):
    """Band-limited state from seeded random physical fields (zero-mean zeta, delta)."""
    rng = np.random.default_rng(seed)
    n = problem.n_grid
    parts = []
    for _ in range(3):
        spec = np.fft.rfft2(amplitude * rng.standard_normal((n, n)))
        spec[~problem.dealias_mask] = 0.0
        parts.append(spec)
    parts[1][0, 0] = 0.0
    parts[2][0, 0] = 0.0
    return np.concatenate([p.ravel() for p in parts])


def main():
    out = {}
    for n in (16, 24, 32, 48, 64, 96):
        prob = PlanarShallowWater(n_grid=n, **PARAMS)
        u = seeded_state(prob, 100 + n, 1e-3)
        out[f"ops_{n}_state"] = u
        out[f"ops_{n}_fe"] = prob.f_expl(u)
        out[f"ops_{n}_fi"] = prob.f_impl(u)
        out[f"ops_{n}_solve"] = prob.implicit_solve(37.5, u)
    prob = PlanarShallowWater(n_grid=32, hyperviscosity=1.0e10, **PARAMS)
    out["ops_32nu_fe"] = prob.f_expl(out["ops_32_state"])

    prob = PlanarShallowWater(n_grid=24, **PARAMS)
    u = jet_initial_condition(prob, JetConfig(perturbation_amplitude=1e-4))
    out["jet24_state"] = u
    cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=4,
                    mode=SweepMode.DIAGONAL_SEQUENTIAL)
    for _ in range(5):
        u, _ = dsdc_step(prob, u, 60.0, cfg)
    out["jet24_dsdc5"] = u

    prob = PlanarShallowWater(n_grid=64, **PARAMS)
    u0 = jet_initial_condition(prob, JetConfig(perturbation_amplitude=1e-2))
    out["jet64_state"] = u0
    cfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=3,
                    mode=SweepMode.DIAGONAL_SEQUENTIAL)
    u = u0
    for _ in range(8):
        u, _ = dsdc_step(prob, u, 120.0, cfg)
    out["jet64_dsdc8"] = u
    scfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=3, mode=SweepMode.SERIAL)
    u = u0
    for _ in range(4):
        u, _ = sdc_step_serial(prob, u, 120.0, scfg)
    out["jet64_serial4"] = u

    prob = PlanarShallowWater(n_grid=32, hyperviscosity=1.0e10, **PARAMS)
    u = seeded_state(prob, 7, 1e-4)
    out["nu32_state"] = u
    for _ in range(3):
        u, _ = dsdc_step(prob, u, 60.0, cfg)
    out["nu32_dsdc3"] = u
    np.savez_compressed(os.path.join(HERE, "planar.npz"), **out)
    print("wrote", os.path.join(HERE, "planar.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
