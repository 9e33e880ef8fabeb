"""Ring output stores, TMA vs plain (SDCSW_RING_TMA_STORE=1/0 in separate runs):
python tools/exp/ring_store_ab.py OUTDIR T:nb[:maxbatch] ...  - saves f_E per case and
prints the live ring stage time; compare two OUTDIRs with --compare A B."""
import os
import sys

import numpy as np

if sys.argv[1] == "--compare":
    a, b = sys.argv[2], sys.argv[3]
    bad = 0
    for f in sorted(os.listdir(a)):
        x, y = np.load(os.path.join(a, f)), np.load(os.path.join(b, f))
        eq = np.array_equal(x.view(np.uint64), y.view(np.uint64))
        bad += not eq
        print(f, "bitwise" if eq else f"DIFF max {np.max(np.abs(x - y)):.3e}")
    sys.exit(1 if bad else 0)

import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2403_20135_b200 import random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

out = sys.argv[1]
os.makedirs(out, exist_ok=True)
mode = os.environ.get("SDCSW_RING_TMA_STORE", "default")
for a in sys.argv[2:]:
    v = [int(x) for x in a.split(":")]
    T, nb = v[0], v[1]
    mb = v[2] if len(v) > 2 else nb
    p = SphericalShallowWater(T, max_batch=mb)
    st = np.stack([random_initial_state(p.grid, s % 8) for s in range(nb)])
    st[:, : p.n_coef] = 3e-3 * st[:, p.n_coef : 2 * p.n_coef] * 1e6
    u = torch.from_numpy(st).to(p.device)
    o = p.empty_states(nb)
    p.f_expl_device(u, o, nb)
    np.save(os.path.join(out, f"T{T}_nb{nb}_mb{mb}.npy"), o.cpu().numpy())
    t = bench.live_stage_times(p, u, reps=20)
    print(f"store={mode} T{T} nb{nb} mb{mb}: ring {t['ring_fft_products'] * 1e6:.1f} us "
          f"synthesis {t['legendre_synthesis'] * 1e6:.1f} analysis {t['legendre_analysis'] * 1e6:.1f}",
          flush=True)
    p.close()
