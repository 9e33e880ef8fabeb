"""Full-length BASELINE configs on the GPU vs the frozen CPU-oracle trajectories.

The golden final states come from tests/golden/make_golden_configs.py: the reference
integrator (parsdc dsdc_step / sdc_step_serial, integrators.py:317-381) driven over the CPU
spherical oracle for the config's full step count. The GPU side is the product path that
bench.py times: the device-resident stepper (fused dSDC step graphs; the 64-member
ensemble batched through the GEMMs for c4). Bar: relative L2 <= 1e-10 per prognostic field
(north star), m > 0 weighted x2.
"""
import os

import numpy as np
import pytest

from oracle.sphere_swe import relative_l2
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-10


class _Weights:
    def __init__(self, trunc):
        from paper_2403_20135_b200.sphere import spectral_index

        self.m_of = spectral_index(trunc)[0]
        self.n_coef = len(self.m_of)


def _load(name):
    path = os.path.join(GOLDEN, f"config_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden trajectory {path} not generated (make_golden_configs.py)")
    return np.load(path)


def _run(name, members_total=1, check_members=None):
    import torch

    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.problem import SphericalShallowWater

    z = _load(name)
    trunc, nodes, sweeps = int(z["trunc"]), int(z["nodes"]), int(z["sweeps"])
    dt, steps, serial = float(z["dt"]), int(z["steps"]), str(z["scheme"]) == "serial"
    seeds = [int(s) for s in z["seeds"]]
    p = SphericalShallowWater(trunc, device=0, max_batch=nodes * members_total)
    cfg = SdcConfig(table=CollocationTable.radau_right(nodes), n_sweeps=sweeps,
                    mode=SweepMode.SERIAL if serial else SweepMode.DIAGONAL_PARALLEL)
    if members_total > 1:
        base = seeds[0]
        u0 = np.stack([random_initial_state(p.grid, base + e) for e in range(members_total)])
        picks = [s - base for s in seeds]
    else:
        u0 = random_initial_state(p.grid, seeds[0])[None]
        picks = [0]
    for i, e in enumerate(picks):
        assert np.isclose(np.sum(np.abs(u0[e])), float(z["u0_abs_sum"][i]), rtol=1e-13, atol=0)
    u = torch.from_numpy(u0).to(p.device).contiguous()
    st = DeviceStepper(p, cfg, dt, serial=serial, members=members_total)
    st.run(u if members_total > 1 else u.reshape(-1), steps, use_graph=True)
    torch.cuda.synchronize()
    assert st.diverged() == 0
    out = u.cpu().numpy()
    w = _Weights(trunc)
    errs = [relative_l2(out[e], z["finals"][i], w) for i, e in enumerate(picks)]
    print(f"{name}: rel L2 per field {errs}")
    st.close()
    p.close()
    return errs


def test_config1_full_200_steps():
    """c1: T127, M=K=4, dt=90 s, 200 steps (the bench workload)."""
    (errs,) = _run("c1")
    assert max(errs) <= TOL, errs


def test_config1_serial_sdc_full_200_steps():
    """c1 as serial SDC (the 1-GPU baseline the speedup is quoted against)."""
    (errs,) = _run("c1s")
    assert max(errs) <= TOL, errs


def test_config2_full_100_steps():
    """c2: T255, M=K=4, dt=60 s, 100 steps."""
    (errs,) = _run("c2")
    assert max(errs) <= TOL, errs


def test_config3_full_50_steps():
    """c3: T511, M=K=5, dt=30 s, 50 steps (table-streaming GEMMs)."""
    (errs,) = _run("c3")
    assert max(errs) <= TOL, errs


def test_config4_ensemble_full_100_steps():
    """c4: all 64 T127 members batched through the GEMMs for 100 steps; members
    0, 31 and 63 against their own oracle trajectories."""
    errs = _run("c4", members_total=64)
    assert max(max(e) for e in errs) <= TOL, errs
