"""A/B timing of node-parallel dSDC over peer memory at world 1 vs the
single-GPU stepper variants (c1 by default)."""
import sys

import torch

from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc
from paper_2403_20135_b200.problem import SphericalShallowWater

T = int(sys.argv[1]) if len(sys.argv) > 1 else 127
M = K = 4
p = SphericalShallowWater(T, max_batch=8)
cfg = SdcConfig(table=CollocationTable.radau_right(M), n_sweeps=K, mode=SweepMode.DIAGONAL_PARALLEL)
u0 = torch.from_numpy(random_initial_state(p.grid, 1)).to(p.device)
u = u0.clone()


def tm(fn, n=200, reps=3):
    fn(8)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(n)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    return best


for fused in (True, False):
    st = DeviceStepper(p, cfg, 90.0, serial=False)
    st.set_fused(fused)
    if not fused:
        st.set_chains(1)
    print(f"stepper fused={fused}: {tm(lambda n: st.run(u, n)):.1f} us/step, launches {st.launches_per_step}")
    st.close()
for fused in (True, False):
    x = PeerNodeParallelDsdc(p, cfg, 90.0, world=1, rank=0, fused=fused)
    print(f"peer fused={fused}: {tm(lambda n: x.run(u, n)):.1f} us/step, launches {x.info()[2]}")
    x.close()
