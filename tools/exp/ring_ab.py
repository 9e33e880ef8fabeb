"""Ring stage time (live states) per truncation for the library in SDCSW_LIB_PATH:
python tools/exp/ring_ab.py T:nb ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2403_20135_b200 import random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

lib = os.path.basename(os.environ.get("SDCSW_LIB_PATH", "default"))
for a in sys.argv[1:]:
    T, nb = (int(x) for x in a.split(":"))
    p = SphericalShallowWater(T, max_batch=nb)
    st = np.stack([random_initial_state(p.grid, s % 8) for s in range(nb)])
    st[:, : p.n_coef] = 3e-3 * st[:, p.n_coef : 2 * p.n_coef] * 1e6
    u = torch.from_numpy(st).to(p.device)
    t = bench.live_stage_times(p, u, reps=20)
    o = p.empty_states(nb)
    p.f_expl_device(u, o, nb)
    print(f"{lib} T{T} nb{nb}: ring {t['ring_fft_products'] * 1e6:.1f} us  "
          f"|fe| {float(torch.linalg.vector_norm(o)):.15e}", flush=True)
    p.close()
