"""Run N steps of one bench config through the device stepper (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.problem import SphericalShallowWater
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
c = bench.CONFIGS[name]
prob = SphericalShallowWater(c["trunc"], max_batch=c["nodes"])
cfg = SdcConfig(table=CollocationTable.radau_right(c["nodes"]), n_sweeps=c["sweeps"], mode=SweepMode.DIAGONAL_PARALLEL)
st = DeviceStepper(prob, cfg, c["dt"], serial=False)
u = prob._to_device(random_initial_state(prob.grid, 0)).reshape(-1).contiguous()
st.run(u, n, use_graph=False)
torch.cuda.synchronize()
print("ok", st.launches_per_step)
