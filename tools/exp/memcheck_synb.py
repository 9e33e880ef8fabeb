"""Small f_E batches for compute-sanitizer memcheck (bulk synthesis
with a partial last batch block).  Run on the GPU box as
compute-sanitizer --tool memcheck python tools/exp/memcheck_synb.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2403_20135_b200 import random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

for nb in (8, 25):
    p = SphericalShallowWater(127, device=0, max_batch=nb)
    st = np.stack([random_initial_state(p.grid, b) for b in range(nb)])
    u = torch.from_numpy(st).to(p.device)
    o = p.empty_states(nb)
    p.f_expl_device(u, o, nb)
    torch.cuda.synchronize()
    print(f"nb={nb} finite={bool(torch.isfinite(torch.view_as_real(o)).all())}", flush=True)
    p.close()
