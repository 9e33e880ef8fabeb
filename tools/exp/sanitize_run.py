"""Small workloads for compute-sanitizer: fused dSDC (T63, T127), unfused/ensemble,
serial SDC, planar, TMA-free paths; a few steps each."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.problem import SphericalShallowWater
from paper_2403_20135_b200.planar import PlanarShallowWater, jet_initial_condition

for T, M in ((63, 3), (127, 4)):
    p = SphericalShallowWater(T, max_batch=8)
    u0 = random_initial_state(p.grid, 1)
    for serial in (False, True):
        mode = SweepMode.SERIAL if serial else SweepMode.DIAGONAL_PARALLEL
        cfg = SdcConfig(table=CollocationTable.radau_right(M), n_sweeps=M, mode=mode)
        st = DeviceStepper(p, cfg, 90.0, serial=serial)
        u = p._to_device(u0).reshape(-1).contiguous()
        st.run(u, 2, use_graph=False)
        if not serial:
            st.set_fused(False); st.set_chains(2); st.run(u, 1, use_graph=False)
        torch.cuda.synchronize(); st.close()
    cfg = SdcConfig(table=CollocationTable.radau_right(M), n_sweeps=M, mode=SweepMode.DIAGONAL_PARALLEL)
    ens = torch.from_numpy(np.stack([u0, u0])).to(p.device).contiguous()
    st = DeviceStepper(p, cfg, 90.0, serial=False, members=2)
    st.run(ens, 1, use_graph=False); torch.cuda.synchronize(); st.close()
    big = p.empty_states(8); src = torch.from_numpy(np.stack([u0] * 8)).to(p.device).contiguous()
    p.f_expl_device(src, big, 8)
    p.close()
pl = PlanarShallowWater(64, 4.0e6, 1.0e5, 1.0e-4, max_batch=4)
x = jet_initial_condition(pl)
cfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=3, mode=SweepMode.DIAGONAL_PARALLEL)
st = DeviceStepper(pl, cfg, 60.0, serial=False)
u = pl._to_device(x).reshape(-1).contiguous(); st.run(u, 2, use_graph=False); torch.cuda.synchronize()
print("sanitize workload done")
