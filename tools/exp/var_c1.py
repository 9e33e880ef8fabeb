"""c1 ring stage + step rate for the library in SDCSW_LIB_PATH (variant sweeps):
python tools/exp/var_c1.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state  # noqa: E402
from paper_2403_20135_b200.integrators import DeviceStepper  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

c = bench.CONFIGS["c1"]
p = SphericalShallowWater(127, max_batch=int(os.environ.get("MAXB", "4")))
cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=4, mode=SweepMode.DIAGONAL_PARALLEL)
st = DeviceStepper(p, cfg, 90.0, serial=False)
u0 = p._to_device(random_initial_state(p.grid, 1)).reshape(-1).contiguous()
u = u0.clone()
st.run(u, 20)
seq = bench.live_states(st, u, 4)
t1 = bench.live_stage_times(p, seq[0].reshape(1, -1).contiguous())
t4 = bench.live_stage_times(p, torch.stack(seq).contiguous())
best = 1e9
for _ in range(5):
    x = u0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.run(x, 200)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 200 * 1e3)
ref = None
lib = os.environ.get("SDCSW_LIB_PATH", "default")
print(f"{os.path.basename(lib)}: ring nb1 {t1['ring_fft_products']*1e6:.2f} nb4 {t4['ring_fft_products']*1e6:.2f} us; "
      f"syn {t1['legendre_synthesis']*1e6:.2f}/{t4['legendre_synthesis']*1e6:.2f}; step {best:.2f} us; "
      f"|u| {float(torch.linalg.vector_norm(x)):.15e}", flush=True)
