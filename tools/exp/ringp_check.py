"""k_ringp (persistent, bulk-prefetched) vs k_ring (one-shot): f_E agreement and the
ring stage time on live-like states.  python tools/exp/ringp_check.py [T ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2403_20135_b200 import random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

for T in [int(a) for a in sys.argv[1:]] or [63, 127, 255, 511]:
    nbs = tuple(int(x) for x in os.environ['NBS'].split()) if 'NBS' in os.environ else ((1, 5) if T >= 400 else (1, 4))
    res = {}
    for r2 in (0, 1):
        os.environ["SDCSW_RINGP"] = str(r2)
        p = SphericalShallowWater(T, device=0, max_batch=max(nbs))
        st = np.stack([random_initial_state(p.grid, s) for s in range(max(nbs))])
        st[:, : p.n_coef] = 3e-3 * st[:, p.n_coef : 2 * p.n_coef] * 1e6
        u = torch.from_numpy(st).to(p.device)
        for nb in nbs:
            o = p.empty_states(nb)
            p.f_expl_device(u[:nb].contiguous(), o, nb)
            torch.cuda.synchronize()
            res[(r2, nb)] = o.cpu().numpy()
            t = bench.live_stage_times(p, u[:nb].contiguous(), reps=20)
            print(f"T{T} ringp={r2} nb={nb}: ring {t['ring_fft_products'] * 1e6:8.2f} us  "
                  f"syn {t['legendre_synthesis'] * 1e6:8.2f} ana {t['legendre_analysis'] * 1e6:8.2f}", flush=True)
        p.close()
    for nb in nbs:
        a, b = res[(0, nb)], res[(1, nb)]
        c = a.shape[1] // 3
        print(f"T{T} nb={nb}: bitwise {np.array_equal(a, b)}", flush=True)
        rel = [np.linalg.norm(a[:, f * c:(f + 1) * c] - b[:, f * c:(f + 1) * c]) /
               np.linalg.norm(a[:, f * c:(f + 1) * c]) for f in range(3)]
        print(f"T{T} nb={nb}: rel per field {['%.2e' % x for x in rel]}", flush=True)
