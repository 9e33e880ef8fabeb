#!/usr/bin/env python
"""Synthesis / analysis stage times (H-free plans) for a knob variant build:
SDCSW_LIB_PATH=build/var/X.so python tools/exp/gemm_knobs.py NAME"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from bench import time_stage  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

name = sys.argv[1]
for T, mb, nbs in ((127, 256, (64, 256)), (255, 4, (1, 4)), (511, 5, (1, 5))):
    p = SphericalShallowWater(T, device=0, max_batch=mb)
    out = []
    for nb in nbs:
        s = min(time_stage(p, 3, nb, reps=10) for _ in range(3)) * 1e6
        a = min(time_stage(p, 2, nb, reps=10) for _ in range(3)) * 1e6
        out.append(f"nb{nb}: syn {s:.1f} ana {a:.1f}")
    print(name, f"T{T}", " | ".join(out), flush=True)
    p.close()
