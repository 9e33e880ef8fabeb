#!/usr/bin/env python
"""Freeze full-length BASELINE-config trajectories of the CPU oracle as golden vectors.

Test infrastructure only. Run in the build container (slow: about an hour for c3):

    python tests/golden/make_golden_configs.py [c1 c1s c2 c3 c4]

For each BASELINE.json config the seeded initial state (bench.py CONFIGS seeds, SURVEY 8(d)
draw order) is advanced for the config's full step count by the REFERENCE integrator
(`parsdc.integrators.dsdc_step`, integrators.py:347-381, or `sdc_step_serial`,
:317-344, for "c1s") over the CPU spherical oracle (oracle/sphere_swe.py). When
/root/reference is absent the bit-identical restatement oracle/sdc.py is used instead
(pinned by sphere_steps.npz). Output: tests/golden/config_<name>.npz with the final state,
the initial-state checksum and the run parameters. c4 freezes members 0, 31 and 63 of
the 64-member ensemble (seeds 100 + member).

The GPU tests (`tests/test_gpu_configs.py`) integrate the same configs on the device and
compare the final states with these at relative L2 <= 1e-10 per field.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.sphere_swe import SphericalShallowWaterOracle  # noqa: E402
from paper_2403_20135_b200.sphere import grid_for, random_initial_state  # noqa: E402

# same table as bench.py CONFIGS (BASELINE.json configs[0..4])
CONFIGS = {
    "c1": dict(trunc=127, nodes=4, sweeps=4, dt=90.0, steps=200, seeds=[1], scheme="dsdc"),
    "c1s": dict(trunc=127, nodes=4, sweeps=4, dt=90.0, steps=200, seeds=[1], scheme="serial"),
    "c2": dict(trunc=255, nodes=4, sweeps=4, dt=60.0, steps=100, seeds=[2], scheme="dsdc"),
    "c3": dict(trunc=511, nodes=5, sweeps=5, dt=30.0, steps=50, seeds=[3], scheme="dsdc"),
    "c4": dict(trunc=127, nodes=4, sweeps=4, dt=90.0, steps=100, seeds=[100, 131, 163],
               scheme="dsdc"),
}


def _stepper(scheme, nodes, sweeps):
    ref = "/root/reference/pkg/src"
    if os.path.isdir(ref):
        sys.path.insert(0, ref)
        from parsdc.collocation import CollocationTable
        from parsdc.integrators import SdcConfig, SweepMode, dsdc_step, sdc_step_serial

        table = CollocationTable.radau_right(nodes)
        if scheme == "dsdc":
            cfg = SdcConfig(table=table, n_sweeps=sweeps, mode=SweepMode.DIAGONAL_SEQUENTIAL)
            return (lambda p, u, dt: dsdc_step(p, u, dt, cfg)[0]), "reference parsdc.dsdc_step"
        cfg = SdcConfig(table=table, n_sweeps=sweeps, mode=SweepMode.SERIAL)
        return (lambda p, u, dt: sdc_step_serial(p, u, dt, cfg)[0]), "reference parsdc.sdc_step_serial"
    from oracle import sdc as osdc
    from paper_2403_20135_b200 import CollocationTable

    table = CollocationTable.radau_right(nodes)
    if scheme == "dsdc":
        return (lambda p, u, dt: osdc.dsdc(p, u, dt, table, sweeps)), "oracle/sdc.py dsdc"
    return (lambda p, u, dt: osdc.serial_sdc(p, u, dt, table, sweeps)), "oracle/sdc.py serial_sdc"


def run(name):
    c = CONFIGS[name]
    g = grid_for(c["trunc"])
    prob = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)
    step, how = _stepper(c["scheme"], c["nodes"], c["sweeps"])
    finals, sums = [], []
    t0 = time.time()
    for seed in c["seeds"]:
        u = random_initial_state(g, seed)
        sums.append(np.sum(np.abs(u)))
        for i in range(c["steps"]):
            u = step(prob, u, c["dt"])
            if not np.isfinite(u).all():
                raise RuntimeError(f"{name}: non-finite at step {i}")
        finals.append(u)
        print(f"{name} seed {seed}: {c['steps']} steps in {time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(
        os.path.join(HERE, f"config_{name}.npz"),
        finals=np.array(finals), seeds=np.array(c["seeds"]), u0_abs_sum=np.array(sums),
        trunc=c["trunc"], nodes=c["nodes"], sweeps=c["sweeps"], dt=c["dt"], steps=c["steps"],
        scheme=c["scheme"], integrator=how,
    )


if __name__ == "__main__":
    for name in sys.argv[1:] or list(CONFIGS):
        run(name)
