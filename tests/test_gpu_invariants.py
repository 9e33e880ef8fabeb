"""Conservation of mass, energy, angular momentum and potential enstrophy over full
BASELINE runs on the GPU path (device-resident dSDC stepper, the path bench.py times),
measured with the CPU oracle's grid diagnostics (tests/sphere_invariants.py).  An
independent check of the spherical operator over its whole spectrum, m > 0 included:
tests/test_invariants.py shows that a wrong sign in any term of the wind synthesis or of
the divergence / curl analysis exceeds these bounds by orders of magnitude within 6 steps.
c2 runs the table-streaming plan (H-free transforms, H-free node kernel)."""

import numpy as np
import pytest

from oracle.sphere_swe import SphericalShallowWaterOracle
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from sphere_invariants import BOUNDS, drifts

pytestmark = pytest.mark.gpu

# BASELINE.json configs c0, c1, c2: (trunc, nodes = sweeps, dt, steps)
_RUNS = {"c0": (63, 3, 120.0, 100), "c1": (127, 4, 90.0, 200), "c2": (255, 4, 60.0, 100)}


@pytest.mark.parametrize("name", sorted(_RUNS))
def test_full_run_conserves_the_invariants(name):
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.problem import SphericalShallowWater

    trunc, nodes, dt, steps = _RUNS[name]
    p = SphericalShallowWater(trunc, device=0, max_batch=nodes)
    assert p.uses_ponly == (trunc >= 200)
    g = p.grid
    o = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)
    u0 = random_initial_state(g, seed=11)
    cfg = SdcConfig(table=CollocationTable.radau_right(nodes), n_sweeps=nodes,
                    mode=SweepMode.DIAGONAL_PARALLEL)
    st = DeviceStepper(p, cfg, dt, serial=False)
    u = torch.from_numpy(u0).to(p.device).reshape(-1).contiguous()
    st.run(u, steps, use_graph=True)
    torch.cuda.synchronize()
    assert st.diverged() == 0
    out = u.cpu().numpy()
    st.close()
    p.close()
    assert np.isfinite(out).all() and not np.array_equal(out, u0)
    d = drifts(o, u0, out)
    print(f"{name}: drifts {d}")
    for k, bound in BOUNDS.items():
        assert d[k] <= bound, (k, d)
