"""A few planar dSDC steps (no CPU leg) for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode  # noqa: E402
from paper_2403_20135_b200.integrators import DeviceStepper  # noqa: E402
from paper_2403_20135_b200.planar import JetConfig, PlanarShallowWater, jet_initial_condition  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
prob = PlanarShallowWater(n, 4.0e6, 1.0e5, 1.0e-4, max_batch=4)
u0 = jet_initial_condition(prob, JetConfig(perturbation_amplitude=1e-2))
cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=4, mode=SweepMode.DIAGONAL_PARALLEL)
st = DeviceStepper(prob, cfg, 60.0, serial=False)
u = prob._to_device(u0).reshape(-1).contiguous()
st.run(u, 3, use_graph=False)
torch.cuda.synchronize()
print("ok")
