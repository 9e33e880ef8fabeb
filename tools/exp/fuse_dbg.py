import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.problem import SphericalShallowWater
p = SphericalShallowWater(63, max_batch=8)
for M, K in [(1, 1), (1, 2), (2, 1), (2, 2), (2, 3), (3, 2), (4, 4)]:
    cfg = SdcConfig(table=CollocationTable.radau_right(M), n_sweeps=K, mode=SweepMode.DIAGONAL_PARALLEL)
    u0 = torch.from_numpy(random_initial_state(p.grid, 30 + M)).to(p.device).contiguous()
    st = DeviceStepper(p, cfg, 90.0, serial=False)
    res = {}
    for setup in ("fused", "batched", "chains", "sequential"):
        st.set_chains(1); st.set_sequential(False); st.set_fused(setup == "fused")
        if setup == "chains": st.set_chains(M)
        if setup == "sequential": st.set_sequential(True)
        u = u0.clone(); st.run(u, 1); torch.cuda.synchronize()
        res[setup] = u.cpu().numpy()
    C = p.n_coef
    out = []
    for k in ("batched", "chains", "sequential"):
        d = np.abs(res[k] - res["fused"])
        out.append(f"{k}: eq={np.array_equal(res[k], res['fused'])} maxd/field=" + ",".join(f"{d[i*C:(i+1)*C].max():.2e}" for i in range(3)))
    print(M, K, "; ".join(out), flush=True)
    st.close()
