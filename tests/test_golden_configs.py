"""CPU checks of the frozen full-length config trajectories (tests/golden/config_*.npz):
parameters match bench.py's CONFIGS (BASELINE.json configs) and the seeded initial states
reproduce (the GPU tests start from the same states)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402
from paper_2403_20135_b200.sphere import grid_for, random_initial_state  # noqa: E402

NAMES = {"c1": "c1", "c1s": "c1", "c2": "c2", "c3": "c3", "c4": "c4"}


@pytest.mark.parametrize("name", sorted(NAMES))
def test_golden_config_matches_bench(name):
    path = os.path.join(ROOT, "tests", "golden", f"config_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_golden_configs.py {name})")
    z = np.load(path)
    c = CONFIGS[NAMES[name]]
    assert (int(z["trunc"]), int(z["nodes"]), int(z["sweeps"])) == (c["trunc"], c["nodes"], c["sweeps"])
    assert (float(z["dt"]), int(z["steps"])) == (c["dt"], c["steps"])
    assert int(z["seeds"][0]) == c["seed"]
    assert str(z["scheme"]) == ("serial" if name == "c1s" else "dsdc")
    finals = z["finals"]
    assert np.isfinite(finals).all() and finals.shape[1] == 3 * (c["trunc"] + 1) * (c["trunc"] + 2) // 2


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_golden_initial_states_reproduce(name):
    z = np.load(os.path.join(ROOT, "tests", "golden", f"config_{name}.npz"))
    g = grid_for(int(z["trunc"]))
    for seed, s in zip(z["seeds"], z["u0_abs_sum"]):
        assert np.isclose(np.sum(np.abs(random_initial_state(g, int(seed)))), float(s), rtol=1e-13, atol=0)
