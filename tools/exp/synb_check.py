"""Bulk-staged GEMM kernels vs the previous ones: f_E agreement and stage times.

python tools/exp/synb_check.py [T ...]   (GPU; KNOB=SDCSW_SYN_BULK (default) or SDCSW_ANA_BULK
selects which kernel is switched per plan; STAGE=3 synthesis, 2 analysis)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from bench import time_stage  # noqa: E402
from paper_2403_20135_b200 import random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

for T in [int(a) for a in sys.argv[1:]] or [127, 255, 511]:
    nbs = tuple(int(x) for x in os.environ["NBS"].split()) if "NBS" in os.environ else (
        (1, 4, 5) if T >= 400 else (1, 4))
    res = {}
    for bulk in (0, 1):
        os.environ[os.environ.get("KNOB", "SDCSW_SYN_BULK")] = str(bulk)
        nmax = max(max(nbs), 6)
        p = SphericalShallowWater(T, device=0, max_batch=nmax)
        st = np.stack([random_initial_state(p.grid, s % 6) for s in range(nmax)])
        st[:, : p.n_coef] = 3e-3 * st[:, p.n_coef : 2 * p.n_coef] * 1e6
        u = torch.from_numpy(st).to(p.device)
        for nb in nbs:
            o = p.empty_states(nb)
            p.f_expl_device(u[:nb].contiguous(), o, nb)
            torch.cuda.synchronize()
            res[(bulk, nb)] = o.cpu().numpy()
            t = time_stage(p, int(os.environ.get("STAGE", "3")), nb, reps=20)
            print(f"T{T} bulk={bulk} nb={nb}: stage {t * 1e6:8.1f} us", flush=True)
        p.close()
    for nb in nbs:
        a, b = res[(0, nb)], res[(1, nb)]
        d = np.linalg.norm(a - b) / np.linalg.norm(a)
        print(f"T{T} nb={nb}: bitwise {np.array_equal(a, b)} rel {d:.2e}", flush=True)
