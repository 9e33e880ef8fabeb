"""One ring launch per (T, nb) inside a profiler region, for
ncu --profile-from-start off --set full.  python tools/exp/ring_prof.py T nb [T nb ...]
(VARIANTS: values of the env knob KNOB, e.g. KNOB=SDCSW_PDL VARIANTS="0 1")"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2403_20135_b200 import _native, random_initial_state  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

args = [int(a) for a in sys.argv[1:]] or [127, 4]
variants = os.environ.get("VARIANTS", "0").split()
knob = os.environ.get("KNOB", "SDCSW_RING_VARIANT")
jobs = []
for T, nb in zip(args[::2], args[1::2]):
    for r2 in variants:
        os.environ[knob] = r2
        p = SphericalShallowWater(T, device=0, max_batch=nb)
        st = np.stack([random_initial_state(p.grid, s) for s in range(nb)])
        u = torch.from_numpy(st).to(p.device)
        o = p.empty_states(nb)
        for stage in (0, 1, 2, 1):
            _native.check(p._lib.sdcsw_transform_stage(p.handle, stage, u.data_ptr(), o.data_ptr(), nb, p.stream()))
        jobs.append((p, u, o, nb))
torch.cuda.synchronize()
torch.cuda.profiler.start()
for p, u, o, nb in jobs:
    _native.check(p._lib.sdcsw_transform_stage(p.handle, 1, u.data_ptr(), o.data_ptr(), nb, p.stream()))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
