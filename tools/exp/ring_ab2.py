#!/usr/bin/env python
"""Ring-kernel variant A/B: ring stage time per (T, nb) and f_E of a seeded state
(saved for the comparison against the default build).

usage: SDCSW_LIB_PATH=build/var/X.so python tools/exp/ring_ab2.py NAME T[:nb,nb..] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from bench import time_stage  # noqa: E402
from paper_2403_20135_b200 import random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

name = sys.argv[1]
os.makedirs("gpurun_out/ab", exist_ok=True)
for spec in sys.argv[2:]:
    T, nbs = spec.split(":")
    T = int(T)
    nbs = [int(x) for x in nbs.split(",")]
    p = SphericalShallowWater(T, device=0, max_batch=max(nbs))
    u = random_initial_state(p.grid, seed=7)
    np.save(f"gpurun_out/ab/fe_{name}_{T}.npy", p.f_expl(u))
    ts = []
    for nb in nbs:
        best = min(time_stage(p, 1, nb, reps=20) for _ in range(3))
        ts.append(f"nb{nb}={best * 1e6:.1f}")
    print(name, f"T{T}", "ring", " ".join(ts), flush=True)
    p.close()
