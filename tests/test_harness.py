"""Harness configuration (CPU) and the GPU CLI path (mirrors
pkg/tests/test_bench_config.py and test_bench_harness.py)."""

import json
import os
import subprocess
import sys

import pytest

from paper_2403_20135_b200.errors import ConfigError
from paper_2403_20135_b200.harness import load_config
from paper_2403_20135_b200.perfmodel import PerfModel, fit_costs, perf_report, theoretical_speedup
from paper_2403_20135_b200.integrators import StepReport

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = """
[problem]
kind = "sphere-swe"
trunc = 63
seed = 2
[stepper]
scheme = "{scheme}"
n_nodes = 3
n_sweeps = 3
dt = 120.0
[run]
t_end = {t_end}
"""


def write(tmp_path, text, name="c.toml"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_load_example():
    cfg = load_config(os.path.join(ROOT, "examples", "t127_dsdc.toml"))
    assert cfg.n_steps() == 200 and cfg.trunc == 127 and len(cfg.candidates) == 2


@pytest.mark.parametrize("bad", [
    SMALL.format(scheme="rk4", t_end=1200.0),
    SMALL.format(scheme="dsdc", t_end=1000.0),  # dt does not divide t_end
    SMALL.replace("sphere-swe", "planar-swe").format(scheme="dsdc", t_end=1200.0),
    "[problem]\nkind='sphere-swe'\n",
])
def test_config_errors(tmp_path, bad):
    with pytest.raises(ConfigError):
        load_config(write(tmp_path, bad))


def test_cli_exit_code_on_bad_config(tmp_path):
    path = write(tmp_path, SMALL.format(scheme="rk4", t_end=1200.0))
    r = subprocess.run([sys.executable, "-m", "paper_2403_20135_b200.cli", "run", "--config", path,
                        "--out", str(tmp_path / "o")], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 2


def test_perfmodel_matches_reference_formulas(reference):
    from parsdc import perfmodel as rp

    for m in (2, 3, 4, 5):
        for r in (0.0, 0.3):
            assert theoretical_speedup(m, r) == rp.theoretical_speedup(m, r)
    reps = [StepReport(1.0, 0.01 + 1e-4 * i, (0.05, 0.05, 0.05), 0.02, 0, 0, 0) for i in range(4)]
    ref_reps = [rp.__dict__ and __import__("parsdc").integrators.StepReport(**r.__dict__) for r in reps]
    a, b = fit_costs(reps, 4), rp.fit_costs(ref_reps, 4)
    assert (a.c_e, a.c_s, a.n_sweeps) == (b.c_e, b.c_s, b.n_sweeps)
    assert perf_report(a, 2.0) == rp.perf_report(b, 2.0)
    assert PerfModel(4, 4, 1.0, 1.0).c_tilde_e == 0.0


@pytest.mark.gpu
def test_cli_run_speedup_perf_model(tmp_path):
    path = write(tmp_path, SMALL.format(scheme="dsdc", t_end=1200.0) +
                 '\n[[speedup.candidate]]\nscheme = "sdc-serial"\ndt = 120.0\n')
    out = tmp_path / "o"
    for cmd in ("run", "speedup", "perf-model"):
        r = subprocess.run([sys.executable, "-m", "paper_2403_20135_b200.cli", cmd, "--config", path,
                            "--out", str(out)], cwd=ROOT, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    rep = json.load(open(out / "run_report.json"))
    assert rep["n_steps"] == 10 and rep["counters"]["n_solve"] == 70
    assert rep["final"]["mean_geopotential_anomaly"] == 0.0
    assert (out / "final_state.snap").exists()
    sp = json.load(open(out / "speedup.json"))
    assert sp["rows"][1]["scheme"] == "sdc-serial"
    pm = json.load(open(out / "perf_model.json"))
    assert pm["M"] == 3 and pm["S_theory"] > 1 and pm["c_E"] > 0 and pm["S_measured"] > 0


PLANAR = """
[problem]
kind = "planar-swe"
n_grid = 24
[problem.jet]
perturbation_amplitude = 1e-4
[stepper]
scheme = "dsdc"
n_nodes = 4
n_sweeps = 4
dt = 60.0
[run]
t_end = 300.0
"""


def test_planar_config_defaults(tmp_path, request):
    """The reference's planar-swe kind and defaults (bench/config.py:178-233)."""
    cfg = load_config(write(tmp_path, PLANAR))
    assert cfg.problem_kind == "planar-swe" and cfg.n_steps() == 5
    assert cfg.problem_params == dict(n_grid=24, domain_length=4.0e6, mean_geopotential=1.0e5,
                                      coriolis=1.0e-4, hyperviscosity=0.0)
    assert cfg.jet_params["perturbation_amplitude"] == 1e-4 and cfg.jet_params["u_max"] == 80.0
    if os.path.isdir("/root/reference/pkg/src"):
        parsdc = request.getfixturevalue("reference")
        from parsdc.bench.config import load_config as ref_load

        ref = ref_load(write(tmp_path, PLANAR, "r.toml"))
        assert ref.problem_params == cfg.problem_params
        assert {k: v for k, v in ref.jet_params.items()} == cfg.jet_params
        del parsdc


@pytest.mark.gpu
def test_cli_planar_run_matches_reference_vectors(tmp_path):
    import numpy as np

    from oracle.planar_swe import relative_l2_fields
    from paper_2403_20135_b200.snapshot import read_planar_snapshot

    path = write(tmp_path, PLANAR)
    out = tmp_path / "p"
    r = subprocess.run([sys.executable, "-m", "paper_2403_20135_b200.cli", "run", "--config", path,
                        "--out", str(out)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rep = json.load(open(out / "run_report.json"))
    assert rep["grid"] == [24, 24] and rep["counters"]["n_solve"] == 5 * 13
    meta, state = read_planar_snapshot(str(out / "final_state.snap"))
    assert meta["n_grid"] == 24 and meta["time"] == 300.0
    gold = np.load(os.path.join(ROOT, "tests", "golden", "planar.npz"))
    assert max(relative_l2_fields(state, gold["jet24_dsdc5"])) <= 1e-10


WP = """
[problem]
kind = "sphere-swe"
trunc = 63
seed = 3
[stepper]
scheme = "dsdc"
n_nodes = 3
n_sweeps = 3
dt_list = [240.0, 120.0]
[run]
t_end = 960.0
reps = 1
[workprecision]
schemes = ["dsdc", "imex-o2"]
[scaling]
splits = [[1, 1], [1, 3], [2, 1]]
"""


def test_workprecision_scaling_config(tmp_path):
    cfg = load_config(write(tmp_path, WP))
    assert cfg.dt_list == [240.0, 120.0] and cfg.wp_schemes == ["dsdc", "imex-o2"]
    assert cfg.scaling_splits == [(1, 1), (1, 3), (2, 1)] and cfg.reference_scheme == "imex-o2"
    with pytest.raises(ConfigError):
        load_config(write(tmp_path, WP.replace("dt_list = [240.0, 120.0]", "dt_list = [250.0]"), "b.toml"))


@pytest.mark.gpu
def test_cli_work_precision_and_scaling(tmp_path):
    import csv as _csv

    path = write(tmp_path, WP)
    out = tmp_path / "wp"
    for cmd in ("work-precision", "scaling"):
        r = subprocess.run([sys.executable, "-m", "paper_2403_20135_b200.cli", cmd, "--config", path,
                            "--out", str(out)], cwd=ROOT, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    pts = list(_csv.DictReader(open(out / "work_precision.csv")))
    assert [p["scheme"] for p in pts] == ["dsdc", "dsdc", "imex-o2", "imex-o2"]
    err = {(p["scheme"], float(p["dt"])): float(p["error"]) for p in pts}
    # dSDC (M=K=3, order <= 5) is far more accurate than the second-order IMEX at the same dt
    assert err[("dsdc", 120.0)] < err[("imex-o2", 120.0)]
    assert err[("imex-o2", 120.0)] < err[("imex-o2", 240.0)]
    rows = list(_csv.DictReader(open(out / "strong_scaling.csv")))
    status = {(r["space_threads"], r["time_threads"]): r["status"] for r in rows}
    assert status[("1", "1")] == "ok" and status[("1", "3")] == "ok" and status[("device", "fused")] == "ok"
    assert status[("2", "1")].startswith("skipped")
