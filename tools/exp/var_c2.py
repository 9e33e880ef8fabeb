"""c2 (T255) stage times + step rate for the library in SDCSW_LIB_PATH."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state  # noqa: E402
from paper_2403_20135_b200.integrators import DeviceStepper  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

cn = os.environ.get("CFG", "c2")
c = bench.CONFIGS[cn]
p = SphericalShallowWater(c["trunc"], max_batch=c["nodes"])
cfg = SdcConfig(table=CollocationTable.radau_right(c["nodes"]), n_sweeps=c["sweeps"], mode=SweepMode.DIAGONAL_PARALLEL)
st = DeviceStepper(p, cfg, c["dt"], serial=False)
u0 = p._to_device(random_initial_state(p.grid, c["seed"])).reshape(-1).contiguous()
u = u0.clone()
st.run(u, 5)
seq = bench.live_states(st, u, c["nodes"])
tm = bench.live_stage_times(p, torch.stack(seq).contiguous())
best = 1e9
for _ in range(3):
    x = u0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.run(x, 20)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 20 * 1e3)
lib = os.environ.get("SDCSW_LIB_PATH", "default")
print(f"{cn} {os.path.basename(lib)}: " + " ".join(f"{k} {v * 1e6:.1f}" for k, v in tm.items()) +
      f"; step {best:.1f} us; |u| {float(torch.linalg.vector_norm(x)):.15e}", flush=True)
