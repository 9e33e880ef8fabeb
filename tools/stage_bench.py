#!/usr/bin/env python
"""Per-stage device times (CUDA events) of f_E and of a full dSDC step, per config.

usage: python tools/stage_bench.py [c0 c1 c2 c3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state  # noqa: E402
from paper_2403_20135_b200.integrators import DeviceStepper  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402


def main(names):
    for name in names:
        c = bench.CONFIGS[name]
        prob = SphericalShallowWater(c["trunc"], max_batch=c["nodes"])
        out = {}
        for stage, sname in ((3, "synth"), (1, "ring"), (2, "anal")):
            for nb in (1, c["nodes"]):
                out[f"{sname}{nb}"] = bench.time_stage(prob, stage, nb, reps=20) * 1e6
        cfg = SdcConfig(table=CollocationTable.radau_right(c["nodes"]), n_sweeps=c["sweeps"],
                        mode=SweepMode.DIAGONAL_PARALLEL)
        st = DeviceStepper(prob, cfg, c["dt"], serial=False)
        u = prob._to_device(random_initial_state(prob.grid, 0)).reshape(-1).contiguous()
        st.run(u, 3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        st.run(u, n)
        e1.record()
        e1.synchronize()
        step = e0.elapsed_time(e1) / n * 1e3
        print(name, " ".join(f"{k}={v:.1f}" for k, v in out.items()), f"step={step:.1f}us",
              f"steps/s={1e6 / step:.0f}", flush=True)
        st.close()
        prob.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c0", "c1", "c2", "c3"])
