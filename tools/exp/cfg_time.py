"""us/step of the default device stepper for bench configs (and a state checksum)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state  # noqa: E402
from paper_2403_20135_b200.integrators import DeviceStepper  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

for name in sys.argv[1:] or ["c0", "c1", "c2"]:
    c = bench.CONFIGS[name]
    E = c.get("members", 1)
    prob = SphericalShallowWater(c["trunc"], max_batch=c["nodes"] * E)
    cfg = SdcConfig(table=CollocationTable.radau_right(c["nodes"]), n_sweeps=c["sweeps"],
                    mode=SweepMode.DIAGONAL_PARALLEL)
    st = DeviceStepper(prob, cfg, c["dt"], serial=False, members=E)
    import numpy as np
    u0 = torch.from_numpy(np.stack([random_initial_state(prob.grid, c["seed"] + e) for e in range(E)])
                          ).to(prob.device).reshape(E, -1).contiguous()
    if E == 1:
        u0 = u0.reshape(-1)
    u = u0.clone()
    n = c["steps"] if E == 1 else 10
    st.run(u, 16)
    best = 1e9
    for _ in range(3):
        u.copy_(u0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.run(u, n)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    h = hashlib.sha1(u.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"{name}: {best:.1f} us/step  sha={h}", flush=True)
    st.close()
