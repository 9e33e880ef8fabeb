"""bench.py host paths without a GPU: the CPU baseline's batched-field problem
agrees with the oracle (and passes the known-answer flows), the reference arm
prints a complete JSON line whose numbers are the ones it timed and whose
workload string is the GPU arm's, and --plan-only reports the multi-GPU
partitions (VERDICT r1 "Next round" items 1 and 5)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.sphere_swe import SphericalShallowWaterFast, SphericalShallowWaterOracle, relative_l2
from paper_2403_20135_b200.sphere import SphereGrid, random_initial_state

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("trunc,nlat,nlon", [(21, 32, 64), (42, 64, 128)])
def test_fast_cpu_problem_matches_oracle(trunc, nlat, nlon):
    o = SphericalShallowWaterOracle(trunc, nlat, nlon)
    f = SphericalShallowWaterFast(trunc, nlat, nlon, tables=(o.mu, o.w, o.p, o.h, o.m_of, o.n_of))
    g = SphereGrid(trunc=trunc, nlat=nlat, nlon=nlon)
    u = random_initial_state(g, 3)
    u[: o.n_coef] = 3e-3 * u[o.n_coef : 2 * o.n_coef] * 1e6
    assert max(relative_l2(f.f_expl(u), o.f_expl(u), o)) <= 1e-12
    from sphere_kats import field_errors, rossby_haurwitz, tilted_potential

    for x, want in (tilted_potential(o, np.pi / 3), rossby_haurwitz(o)):
        fe, fi = f.f_expl(x), f.f_impl(x)
        assert max(field_errors(o, fe + fi, want, [fe, fi])[:2]) <= 1e-10


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_line():
    line = run_bench("--impl", "reference", "--config", "c0", "--steps", "2", "--warmup", "1")
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["value"] > 0 and abs(line["ms_per_step"] - 1e3 / line["value"]) < 1e-6 * line["ms_per_step"]
    assert line["config"]["workload"].startswith("c0: T63 192x96 M=3 K=3 dt=120.0 s, 100 time steps")
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "steps/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    import bench

    assert line["config"]["workload"] == bench.workload_string("c0", 192, 96)


def test_plan_only():
    out = run_bench("--plan-only")["configs"]
    assert out["c3"]["8"]["node_groups"] == 1 and out["c3"]["8"]["spectral_parts"] == 8
    assert out["c1"]["4"]["node_groups"] == 4 and out["c1"]["4"]["spectral_parts"] == 1
    assert out["c2"]["8"]["node_groups"] == 4 and out["c2"]["8"]["spectral_parts"] == 2
    assert out["c4"]["8"]["members_per_gpu"] == 8
    for n in ("2", "4", "8"):
        c3 = out["c3"][n]
        assert sum(c3["coefficients_per_part"]) == 512 * 513 // 2
