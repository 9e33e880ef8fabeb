#!/usr/bin/env python
"""H-free (P-only) transforms vs the P/H path: f_E agreement and stage times.

usage: python tools/exp/ponly_check.py [T:max_batch:nb ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import time_stage  # noqa: E402
from paper_2403_20135_b200 import random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402


def run(T, mb, nb, po):
    os.environ["SDCSW_PONLY"] = str(po)
    p = SphericalShallowWater(T, device=0, max_batch=mb)
    u = torch.stack([torch.from_numpy(random_initial_state(p.grid, seed=s)) for s in range(nb)]).to(0)
    out = p.empty_states(nb)
    p.f_expl_device(u, out, nb)
    fe = out.cpu().numpy()
    times = {k: min(time_stage(p, st, nb, reps=10) for _ in range(3)) * 1e6
             for k, st in (("synth", 3), ("ring", 1), ("anal", 2))}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        p.f_expl_device(u, out, nb)
    ev0.record()
    for _ in range(10):
        p.f_expl_device(u, out, nb)
    ev1.record()
    ev1.synchronize()
    times["fE"] = ev0.elapsed_time(ev1) / 10 * 1e3
    p.close()
    return fe, times


for spec in sys.argv[1:] or ["127:16:4", "255:4:4", "511:5:5"]:
    T, mb, nb = (int(x) for x in spec.split(":"))
    fa, ta = run(T, mb, nb, 0)
    fb, tb = run(T, mb, nb, 1)
    rel = max(np.linalg.norm(fa[b] - fb[b]) / np.linalg.norm(fa[b]) for b in range(nb))
    C = fa.shape[1] // 3
    relf = [max(np.linalg.norm(fa[b, k * C:(k + 1) * C] - fb[b, k * C:(k + 1) * C])
                / np.linalg.norm(fa[b, k * C:(k + 1) * C]) for b in range(nb)) for k in range(3)]
    print(f"T{T} mb{mb} nb{nb}: rel L2 P-only vs P/H {rel:.2e} per field {['%.1e' % x for x in relf]}")
    print("   P/H   ", " ".join(f"{k}={v:.1f}" for k, v in ta.items()))
    print("   P-only", " ".join(f"{k}={v:.1f}" for k, v in tb.items()), flush=True)
