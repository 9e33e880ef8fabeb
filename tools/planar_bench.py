#!/usr/bin/env python
"""The reference's own problem (planar shallow water, balanced jet) on the GPU
against its CPU implementation restated in oracle/planar_swe.py + oracle/sdc.py
(bit-identical integrator, numpy FFTs as the reference's scipy FFTs).

usage: python tools/planar_bench.py [--n 256] [--nodes 4] [--sweeps 4] [--dt 60] [--steps 100]
Prints one JSON line (not the bench.py contract; an extra data point)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode  # noqa: E402
from paper_2403_20135_b200.integrators import DeviceStepper  # noqa: E402
from paper_2403_20135_b200.planar import JetConfig, PlanarShallowWater, jet_initial_condition  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--nodes", type=int, default=4)
    ap.add_argument("--sweeps", type=int, default=4)
    ap.add_argument("--dt", type=float, default=60.0)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--cpu-steps", type=int, default=2)
    a = ap.parse_args()
    prob = PlanarShallowWater(a.n, 4.0e6, 1.0e5, 1.0e-4, max_batch=a.nodes)
    u0 = jet_initial_condition(prob, JetConfig(perturbation_amplitude=1e-2))
    cfg = SdcConfig(table=CollocationTable.radau_right(a.nodes), n_sweeps=a.sweeps,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=a.nodes)
    st = DeviceStepper(prob, cfg, a.dt, serial=False)
    u = prob._to_device(u0).reshape(-1).contiguous()
    st.run(u, 5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    u.copy_(prob._to_device(u0).reshape(-1))
    e0.record()
    st.run(u, a.steps)
    e1.record()
    e1.synchronize()
    gpu_rate = a.steps / (e0.elapsed_time(e1) * 1e-3)
    st.close()
    # CPU: the reference integrator restated bit-for-bit over the numpy planar problem
    from oracle import sdc as osdc
    from oracle.planar_swe import PlanarShallowWaterOracle

    o = PlanarShallowWaterOracle(a.n, 4.0e6, 1.0e5, 1.0e-4)
    x = u0.copy()
    x = osdc.dsdc(o, x, a.dt, cfg.table, a.sweeps)  # warm-up
    t0 = time.perf_counter()
    for _ in range(a.cpu_steps):
        x = osdc.dsdc(o, x, a.dt, cfg.table, a.sweeps)
    cpu_rate = a.cpu_steps / (time.perf_counter() - t0)
    print(json.dumps({"problem": f"planar-swe N={a.n} balanced jet (the reference's own problem)",
                      "scheme": f"dSDC M={a.nodes} K={a.sweeps} dt={a.dt}",
                      "gpu_steps_per_s": gpu_rate, "cpu_steps_per_s": cpu_rate,
                      "cpu_threads": 1, "cpu_sample_steps": a.cpu_steps,
                      "speedup": gpu_rate / cpu_rate}))


if __name__ == "__main__":
    main()
