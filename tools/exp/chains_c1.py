"""c1 step time: fused batched step (default) vs unfused with 1 / 2 / 4 concurrent node chains."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.problem import SphericalShallowWater

T, M, dt = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (127, 4, 90.0)
p = SphericalShallowWater(T, max_batch=max(8, M))
u0 = random_initial_state(p.grid, 1)
cfg = SdcConfig(table=CollocationTable.radau_right(M), n_sweeps=M, mode=SweepMode.DIAGONAL_PARALLEL)
for label, fused, chains in (("fused", True, 1), ("unfused c1", False, 1), ("unfused c2", False, 2),
                             ("unfused c4", False, M)):
    st = DeviceStepper(p, cfg, dt, serial=False)
    if not fused:
        st.set_fused(False)
        st.set_chains(chains)
    u = p._to_device(u0).reshape(-1).contiguous()
    st.run(u, 40, use_graph=True)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); st.run(u, 200, use_graph=True); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 200 * 1e3)
    print(f"T{T} {label}: {best:.1f} us/step, launches {st.launches_per_step}", flush=True)
    st.close()
