"""A few steps of the unfused stepper and of the world-1 peer exchange (for an ncu launch list)."""
import torch

from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc
from paper_2403_20135_b200.problem import SphericalShallowWater

p = SphericalShallowWater(127, max_batch=8)
cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=4, mode=SweepMode.DIAGONAL_PARALLEL)
u = torch.from_numpy(random_initial_state(p.grid, 1)).to(p.device)
st = DeviceStepper(p, cfg, 90.0, serial=False)
st.set_fused(False)
st.set_chains(1)
st.run(u, 2, use_graph=False)
torch.cuda.synchronize()
x = PeerNodeParallelDsdc(p, cfg, 90.0, world=1, rank=0)
x.run(u, 2, use_graph=False)
torch.cuda.synchronize()
