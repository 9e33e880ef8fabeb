#!/usr/bin/env python
"""Launch each f_E stage a few times at one config (for ncu): python tools/prof_stages.py c1 4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2403_20135_b200 import _native, random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else bench.CONFIGS[name]["nodes"]
c = bench.CONFIGS[name]
p = SphericalShallowWater(c["trunc"], max_batch=max(nb, c["nodes"]))
u = torch.from_numpy(__import__("numpy").stack([random_initial_state(p.grid, s) for s in range(nb)])).to(p.device)
out = p.empty_states(nb)
for rep in range(3):
    for stage in (0, 3, 1, 2):
        _native.check(p._lib.sdcsw_transform_stage(p.handle, stage, u.data_ptr(), out.data_ptr(), nb, p.stream()))
torch.cuda.synchronize()
for stage, nm in ((3, "synth-only"), (1, "ring"), (2, "anal")):
    print(nm, bench.time_stage(p, stage, nb) * 1e6)
