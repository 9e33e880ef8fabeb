#!/usr/bin/env python
"""A/B of the dSDC step variants (fused epilogue / batched / chains) per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state  # noqa: E402
from paper_2403_20135_b200.integrators import DeviceStepper  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402


def timed(st, u, n=200):
    st.run(u, 5)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.run(u, n)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / n * 1e3)
    return best


for name in sys.argv[1:] or ["c0", "c1", "c2"]:
    c = bench.CONFIGS[name]
    prob = SphericalShallowWater(c["trunc"], max_batch=c["nodes"])
    cfg = SdcConfig(table=CollocationTable.radau_right(c["nodes"]), n_sweeps=c["sweeps"],
                    mode=SweepMode.DIAGONAL_PARALLEL)
    st = DeviceStepper(prob, cfg, c["dt"], serial=False)
    u = prob._to_device(random_initial_state(prob.grid, 0)).reshape(-1).contiguous()
    res = {}
    for setup in ("fused", "batched", "chains2", "chainsM"):
        try:
            st.set_chains(1)
            st.set_fused(setup == "fused")
            if setup == "chains2":
                st.set_chains(min(2, c["nodes"]))
            if setup == "chainsM":
                st.set_chains(c["nodes"])
        except Exception as exc:  # noqa: BLE001
            res[setup] = str(exc)[:30]
            continue
        res[setup] = f"{timed(st, u):.1f}us/{st.launches_per_step}"
    print(name, res, flush=True)
