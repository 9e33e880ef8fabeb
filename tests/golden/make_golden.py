#!/usr/bin/env python
"""Generate the committed golden vectors from the READ-ONLY reference package.

Run in the build container (the reference is mounted at /root/reference):

    python tests/golden/make_golden.py

Outputs (small .npz files in tests/golden/):
  collocation.npz  Radau-right nodes / Q / dtau for M = 1..16 and MIN-SR-FLEX
                   diagonals, from parsdc.collocation (collocation.py:117-256)
  dahlquist.npz    reference dsdc_step / sdc_step_serial results and evaluation
                   counts on parsdc's own DahlquistProblem (integrators.py:317-381)
  sphere_steps.npz reference dsdc_step / sdc_step_serial / integrate driven over
                   the CPU spherical oracle (T21, 64x32), plus the seeded initial
                   state: pins oracle/sdc.py bit-for-bit against the reference
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from parsdc import collocation as rc  # noqa: E402
from parsdc.integrators import (  # noqa: E402
    Ab2SiStepper,
    DiagonalSdcStepper,
    ImexO2Stepper,
    SdcConfig,
    SerialSdcStepper,
    SweepMode,
    dsdc_step,
    integrate,
    sdc_step_serial,
)
from parsdc.problems import DahlquistProblem  # noqa: E402

from oracle.sphere_swe import SphericalShallowWaterOracle  # noqa: E402
from paper_2403_20135_b200.sphere import SphereGrid, random_initial_state  # noqa: E402


def collocation():
    out = {}
    for m in range(1, rc.MAX_NODES + 1):
        t = rc.CollocationTable.radau_right(m)
        out[f"nodes_{m}"] = t.nodes
        out[f"q_{m}"] = t.q_matrix
        out[f"dtau_{m}"] = t.dtau
        for k in (1, 2, 3, 4):
            out[f"minsr_{m}_{k}"] = rc.diagonal_coefficients(rc.DiagonalPreconditioner.MIN_SR_FLEX, t, k)
    np.savez_compressed(os.path.join(HERE, "collocation.npz"), **out)


def dahlquist():
    out = {}
    prob = DahlquistProblem(lambda_impl=-1.0 + 0.3j, lambda_expl=0.2j, width=3)
    u0 = np.array([1.0 + 0j, 0.5 - 0.25j, -2.0 + 1j])
    for m, k in ((2, 2), (3, 3), (4, 4), (5, 5), (4, 1)):
        table = rc.CollocationTable.radau_right(m)
        cfg = SdcConfig(table=table, n_sweeps=k, mode=SweepMode.DIAGONAL_SEQUENTIAL)
        prob.reset_counters()
        u, rep = dsdc_step(prob, u0, 0.3, cfg)
        out[f"dsdc_{m}_{k}"] = u
        out[f"dsdc_counts_{m}_{k}"] = np.array([rep.n_f_expl, rep.n_f_impl, rep.n_solve])
        cfg = SdcConfig(table=table, n_sweeps=k, mode=SweepMode.SERIAL)
        prob.reset_counters()
        u, rep = sdc_step_serial(prob, u0, 0.3, cfg)
        out[f"serial_{m}_{k}"] = u
        out[f"serial_counts_{m}_{k}"] = np.array([rep.n_f_expl, rep.n_f_impl, rep.n_solve])
    out["u0"] = u0
    np.savez_compressed(os.path.join(HERE, "dahlquist.npz"), **out)


def sphere_steps():
    grid = SphereGrid(trunc=21, nlat=32, nlon=64)
    prob = SphericalShallowWaterOracle(grid.trunc, grid.nlat, grid.nlon)
    u0 = random_initial_state(grid, seed=11)
    out = {"u0": u0}
    for m, k in ((3, 3), (4, 4)):
        table = rc.CollocationTable.radau_right(m)
        cfg = SdcConfig(table=table, n_sweeps=k, mode=SweepMode.DIAGONAL_SEQUENTIAL)
        out[f"dsdc_{m}_{k}"] = dsdc_step(prob, u0, 600.0, cfg)[0]
        cfg = SdcConfig(table=table, n_sweeps=k, mode=SweepMode.SERIAL)
        out[f"serial_{m}_{k}"] = sdc_step_serial(prob, u0, 600.0, cfg)[0]
    table = rc.CollocationTable.radau_right(3)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.DIAGONAL_PARALLEL, time_threads=3)
    traj = integrate(prob, u0, 600.0, 4, DiagonalSdcStepper(cfg), checkpoint_interval=2)
    cfg.close()
    out["integrate_dsdc_states"] = np.array(traj.states)
    out["integrate_dsdc_times"] = np.array(traj.times)
    cfg = SdcConfig(table=table, n_sweeps=3, mode=SweepMode.SERIAL)
    traj = integrate(prob, u0, 600.0, 3, SerialSdcStepper(cfg))
    out["integrate_serial_final"] = traj.states[-1]
    traj = integrate(prob, u0, 300.0, 3, ImexO2Stepper())
    out["imex_o2_final"] = traj.states[-1]
    out["imex_o2_counts"] = np.array([[r.n_f_expl, r.n_f_impl, r.n_solve] for r in traj.reports])
    traj = integrate(prob, u0, 300.0, 4, Ab2SiStepper())
    out["ab2_si_final"] = traj.states[-1]
    out["ab2_si_counts"] = np.array([[r.n_f_expl, r.n_f_impl, r.n_solve] for r in traj.reports])
    np.savez_compressed(os.path.join(HERE, "sphere_steps.npz"), **out)


if __name__ == "__main__":
    collocation()
    dahlquist()
    sphere_steps()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
