"""Benchmark harness for the GPU path: ``sphere-swe`` TOML configurations.

Mirrors the reference harness (``pkg/src/parsdc/bench/config.py``,
``harness.py``, ``cli.py``) for the spherical problem on
the device:

``[problem]``  ``kind = "sphere-swe"``, ``trunc``, optional ``nlat``/``nlon``
               and physical constants, ``seed`` (seeded BASELINE spectrum,
               SURVEY 8d) or ``initial = "<snapshot path>"``; or the
               reference's ``kind = "planar-swe"`` (``n_grid``, ``domain_length``,
               ``mean_geopotential``, ``coriolis``, ``hyperviscosity``, optional
               ``[problem.jet]``), run on the GPU planar problem.
``[stepper]``  ``scheme`` in {dsdc, sdc-serial, imex-o2, ab2-si}, ``n_nodes``,
               ``n_sweeps``, ``preconditioner`` (min-sr-flex | implicit-euler),
               ``dt``.
``[run]``      ``t_end``, optional ``checkpoint_interval`` (steps), ``reps``.
``[[speedup.candidate]]``  ``scheme`` and ``dt``.

Reports: ``run_report.json`` + ``final_state.snap`` (:mod:`.snapshot`; PSWSNAP1 for planar),
``speedup.json`` / ``speedup.csv``, ``perf_model.json`` (cost model fitted from
CUDA-event stage timings, S_theory vs the measured sequential/parallel ratio).
"""

import csv
import json
import math
import os
import platform
import time

try:
    import tomllib
except ModuleNotFoundError:  # pragma: no cover
    import tomli as tomllib

import numpy as np

from .collocation import MAX_NODES, CollocationTable, DiagonalPreconditioner
from .core import evaluation_counters, state_norm
from .errors import ConfigError, ParameterError
from .integrators import (
    DeviceStepper,
    DiagonalSdcStepper,
    SdcConfig,
    SerialSdcStepper,
    SweepMode,
    integrate,
)
from .perfmodel import fit_costs, perf_report

SCHEMES = ("dsdc", "sdc-serial", "imex-o2", "ab2-si")
_PRECOND = {"min-sr-flex": DiagonalPreconditioner.MIN_SR_FLEX,
            "implicit-euler": DiagonalPreconditioner.IMPLICIT_EULER_DTAU}


class ExperimentConfig:
    """Validated contents of one TOML file (ConfigError on any violation)."""

    def __init__(self, data):
        def get(section, key, default=None, required=False):
            sec = data.get(section, {})
            if key not in sec:
                if required:
                    raise ConfigError(f"[{section}] {key} is required")
                return default
            return sec[key]

        self.title = data.get("title", "")
        kind = get("problem", "kind", required=True)
        if kind not in ("sphere-swe", "planar-swe"):
            raise ConfigError(f"problem kind must be 'sphere-swe' or 'planar-swe', got {kind!r}")
        self.problem_kind = kind
        self.jet_params = {}
        if kind == "sphere-swe":
            self.trunc = int(get("problem", "trunc", required=True))
            if self.trunc < 1:
                raise ConfigError("trunc must be positive")
            self.problem_params = {k: get("problem", k) for k in
                                   ("nlat", "nlon", "radius", "gravity", "omega", "mean_depth")
                                   if get("problem", k) is not None}
        else:  # the reference's planar kind and defaults (bench/config.py:178-233)
            self.trunc = None
            self.problem_params = {
                "n_grid": int(get("problem", "n_grid", required=True)),
                "domain_length": float(get("problem", "domain_length", 4.0e6)),
                "mean_geopotential": float(get("problem", "mean_geopotential", 1.0e5)),
                "coriolis": float(get("problem", "coriolis", 1.0e-4)),
                "hyperviscosity": float(get("problem", "hyperviscosity", 0.0)),
            }
            if self.problem_params["n_grid"] < 1 or self.problem_params["domain_length"] <= 0 \
                    or self.problem_params["mean_geopotential"] <= 0:
                raise ConfigError("planar-swe needs positive n_grid, domain_length, mean_geopotential")
            jet = data.get("problem", {}).get("jet", {})
            if not isinstance(jet, dict):
                raise ConfigError("[problem.jet] must be a table")
            self.jet_params = {
                "u_max": float(jet.get("u_max", 80.0)),
                "perturbation_amplitude": float(jet.get("perturbation_amplitude", 1.0e-4)),
                "perturbation_wavenumber": int(jet.get("perturbation_wavenumber", 3)),
            }
            for opt in ("y_center", "width"):
                if opt in jet:
                    self.jet_params[opt] = float(jet[opt])
        self.seed = int(get("problem", "seed", 0))
        self.initial = get("problem", "initial")
        self.scheme = get("stepper", "scheme", required=True)
        if self.scheme not in SCHEMES:
            raise ConfigError(f"scheme must be one of {SCHEMES}, got {self.scheme!r}")
        self.n_nodes = int(get("stepper", "n_nodes", 3))
        if not 1 <= self.n_nodes <= MAX_NODES:
            raise ConfigError(f"n_nodes must be in [1, {MAX_NODES}]")
        self.n_sweeps = int(get("stepper", "n_sweeps", self.n_nodes))
        if self.n_sweeps < 1:
            raise ConfigError("n_sweeps must be positive")
        pc = get("stepper", "preconditioner", "min-sr-flex")
        if pc not in _PRECOND:
            raise ConfigError(f"unknown preconditioner {pc!r}")
        self.preconditioner = _PRECOND[pc]
        dt = get("stepper", "dt")
        dt_list = get("stepper", "dt_list")
        if dt is None and dt_list is None:
            raise ConfigError("[stepper] needs 'dt' or 'dt_list'")
        if dt_list is not None:
            if not isinstance(dt_list, list) or not dt_list or not all(
                    isinstance(v, (int, float)) and not isinstance(v, bool) and v > 0 for v in dt_list):
                raise ConfigError("stepper.dt_list must be a non-empty list of positive step sizes")
            dt_list = [float(v) for v in dt_list]
        self.dt = float(dt if dt is not None else dt_list[0])
        self.dt_list = dt_list if dt_list is not None else [self.dt]
        self.t_end = float(get("run", "t_end", required=True))
        if self.dt <= 0 or self.t_end <= 0:
            raise ConfigError("dt and t_end must be positive")
        # work-precision / scaling sections (reference bench/config.py:296-340)
        self.metric = data.get("metric", {}).get("kind", "rel")
        if self.metric not in ("rel", "abs"):
            raise ConfigError(f"metric must be 'rel' or 'abs', got {self.metric!r}")
        ref = data.get("reference", {})
        self.reference_scheme = ref.get("scheme", "imex-o2")
        if self.reference_scheme not in SCHEMES:
            raise ConfigError(f"unknown reference scheme {self.reference_scheme!r}")
        self.reference_dt = float(ref["dt"]) if "dt" in ref else None
        self.wp_schemes = data.get("workprecision", {}).get("schemes", [self.scheme])
        for name in self.wp_schemes:
            if name not in SCHEMES:
                raise ConfigError(f"unknown scheme {name!r} in workprecision.schemes")
        self.scaling_splits = [tuple(v) for v in data.get("scaling", {}).get("splits", [[1, 1]])]
        for pair in self.scaling_splits:
            if len(pair) != 2 or not all(isinstance(v, int) and v >= 1 for v in pair):
                raise ConfigError(f"scaling.splits entries must be [space, time] positive pairs, got {pair!r}")
        self.checkpoint_interval = get("run", "checkpoint_interval")
        self.reps = int(get("run", "reps", 1))
        self.candidates = [dict(c) for c in data.get("speedup", {}).get("candidate", [])]
        for c in self.candidates:
            if c.get("scheme") not in SCHEMES or float(c.get("dt", 0)) <= 0:
                raise ConfigError(f"bad speedup candidate {c}")
        self.n_steps(self.dt)
        for d in self.dt_list:
            self.n_steps(d)
        for c in self.candidates:
            self.n_steps(float(c["dt"]))

    def n_steps(self, dt=None):
        dt = self.dt if dt is None else dt
        n = self.t_end / dt
        if abs(n - round(n)) > 1e-9 * max(1.0, n):
            raise ConfigError(f"dt = {dt} does not divide t_end = {self.t_end}")
        return int(round(n))


def load_config(path):
    try:
        with open(path, "rb") as f:
            data = tomllib.load(f)
    except (OSError, tomllib.TOMLDecodeError) as exc:
        raise ConfigError(f"cannot read {path}: {exc}") from exc
    return ExperimentConfig(data)


def build_problem(config):
    if config.problem_kind == "planar-swe":
        from .planar import PlanarShallowWater

        return PlanarShallowWater(max_batch=max(8, config.n_nodes), **config.problem_params)
    from .problem import SphericalShallowWater

    return SphericalShallowWater(config.trunc, max_batch=max(8, config.n_nodes),
                                 **config.problem_params)


def build_initial_state(config, problem):
    if config.problem_kind == "planar-swe":
        from .planar import JetConfig, jet_initial_condition

        return jet_initial_condition(problem, JetConfig(**config.jet_params))
    if config.initial:
        from .snapshot import read_snapshot

        meta, state = read_snapshot(config.initial)
        if meta["grid"].trunc != config.trunc:
            raise ConfigError("snapshot truncation does not match the problem")
        return state
    from .sphere import random_initial_state

    return random_initial_state(problem.grid, config.seed)


def build_stepper(config, scheme=None):
    scheme = config.scheme if scheme is None else scheme
    if scheme == "imex-o2":
        from .schemes import ImexO2Stepper

        return ImexO2Stepper()
    if scheme == "ab2-si":
        from .schemes import Ab2SiStepper

        return Ab2SiStepper()
    table = CollocationTable.radau_right(config.n_nodes)
    if scheme == "sdc-serial":
        return SerialSdcStepper(SdcConfig(table=table, n_sweeps=config.n_sweeps, mode=SweepMode.SERIAL))
    return DiagonalSdcStepper(SdcConfig(table=table, n_sweeps=config.n_sweeps,
                                        preconditioner=config.preconditioner,
                                        mode=SweepMode.DIAGONAL_PARALLEL,
                                        time_threads=config.n_nodes))


def environment_info():
    import torch

    from . import __version__

    return {
        "platform": platform.platform(),
        "python": platform.python_version(),
        "torch": torch.__version__,
        "gpu": torch.cuda.get_device_name(0) if torch.cuda.is_available() else None,
        "package": __version__,
    }


def _timed(problem, state, dt, n, stepper, interval=None):
    import torch

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    traj = integrate(problem, state, dt, n, stepper, checkpoint_interval=interval)
    torch.cuda.synchronize()
    return traj, time.perf_counter() - t0


def run_single(config, out_dir):
    """One integration; writes run_report.json and final_state.snap."""
    from .snapshot import write_planar_snapshot, write_snapshot

    os.makedirs(out_dir, exist_ok=True)
    problem = build_problem(config)
    state = build_initial_state(config, problem)
    stepper = build_stepper(config)
    n = config.n_steps()
    try:
        traj, wall = _timed(problem, state, config.dt, n, stepper, config.checkpoint_interval)
    finally:
        if getattr(stepper, "cfg", None) is not None:
            stepper.cfg.close()
    final = traj.states[-1]
    c = problem.n_coef
    walls = [r.wall_s for r in traj.reports]
    planar = config.problem_kind == "planar-swe"
    grid = [problem.n_grid] * 2 if planar else [problem.grid.nlon, problem.grid.nlat]
    mean_phi = problem.mean_geopotential_anomaly(final) if planar else float(final[0].real)
    report = {
        "title": config.title, "problem": config.problem_kind, "scheme": traj.scheme,
        "trunc": config.trunc, "grid": grid, "dt": config.dt,
        "n_steps": n, "t_end": config.t_end, "wall_s": wall,
        "steps_per_s": n / wall,
        "step_wall_s": {"min": min(walls), "median": float(np.median(walls)), "max": max(walls)},
        "counters": dict(zip(("n_f_expl", "n_f_impl", "n_solve"), evaluation_counters(problem))),
        "checkpoint_times": traj.times,
        "final": {"state_norm": state_norm(final),
                  "mean_geopotential_anomaly": mean_phi,
                  "vorticity_norm": float(np.linalg.norm(final[c : 2 * c]))},
        "environment": environment_info(),
    }
    writer = write_planar_snapshot if planar else write_snapshot
    writer(os.path.join(out_dir, "final_state.snap"), problem, final, config.t_end)
    with open(os.path.join(out_dir, "run_report.json"), "w") as f:
        json.dump(report, f, indent=2, sort_keys=True)
    problem.close()
    return report


def _reference_dt(config):
    finest = min(config.dt_list)
    if config.reference_dt is not None:
        if config.reference_dt > finest / 8.0:
            raise ConfigError(f"reference dt {config.reference_dt} coarser than one eighth of the "
                              f"finest candidate dt {finest}")
        return config.reference_dt
    return finest / 64.0


def _aligned_intervals(dts, reference_dt):
    """Checkpoint intervals on multiples of the coarsest dt (None: endpoints only)."""
    coarsest = max(dts)
    out = []
    for dt in list(dts) + [reference_dt]:
        r = coarsest / dt
        if abs(r - round(r)) > 1e-9:
            return [None] * len(dts), None
        out.append(int(round(r)))
    return out[:-1], out[-1]


def work_precision(config, out_dir):
    """Error against wall time per (scheme, dt) - the reference's work-precision
    sweep (``bench/harness.py:228-270``) on the GPU steppers.  Writes
    ``work_precision.csv`` (scheme, dt, wall_s, error, status); errors use
    :func:`.metrics.error_linf_l2` on the vorticity grid field against a fine
    reference trajectory at checkpoints aligned on the coarsest step."""
    from .errors import DivergenceError
    from .metrics import error_linf_l2

    os.makedirs(out_dir, exist_ok=True)
    dts = sorted(config.dt_list, reverse=True)
    ref_dt = _reference_dt(config)
    intervals, ref_interval = _aligned_intervals(dts, ref_dt)
    problem = build_problem(config)
    state = build_initial_state(config, problem)
    ref_stepper = build_stepper(config, config.reference_scheme)
    try:
        reference, _ = _timed(problem, state, ref_dt, config.n_steps(ref_dt), ref_stepper, ref_interval)
    finally:
        if getattr(ref_stepper, "cfg", None) is not None:
            ref_stepper.cfg.close()
    points = []
    for scheme in config.wp_schemes:
        for dt, interval in zip(dts, intervals):
            stepper = build_stepper(config, scheme)
            try:
                traj, wall = _timed(problem, state, dt, config.n_steps(dt), stepper, interval)
                error = error_linf_l2(traj, reference, problem, relative=config.metric == "rel")
                status = "ok"
            except DivergenceError:
                error = wall = float("nan")
                status = "diverged"
            finally:
                if getattr(stepper, "cfg", None) is not None:
                    stepper.cfg.close()
            points.append({"scheme": scheme, "dt": dt, "wall_s": wall, "error": error, "status": status})
    with open(os.path.join(out_dir, "work_precision.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["scheme", "dt", "wall_s", "error", "status"])
        w.writeheader()
        w.writerows(points)
    problem.close()
    return points


def strong_scaling(config, out_dir):
    """Wall time across (space, time) splits - the reference's thread-split sweep
    (``bench/harness.py:273-333``) mapped onto one GPU: the time split is the
    number of concurrent node groups per sweep (1 = one node after another, the
    DIAGONAL_SEQUENTIAL analogue; M = every node on its own graph branch) and
    the space split has no GPU meaning (each row records it; only 1 runs).  A
    "device" row adds the default fused step (all nodes batched into the GEMMs).
    Writes ``strong_scaling.csv`` with the reference's columns."""
    import torch

    os.makedirs(out_dir, exist_ok=True)
    splits = list(config.scaling_splits)
    if (1, 1) not in splits:
        splits.insert(0, (1, 1))
    n = config.n_steps()
    problem = build_problem(config)
    state = build_initial_state(config, problem)
    u0 = problem._to_device(state).reshape(-1).contiguous()
    table = CollocationTable.radau_right(config.n_nodes)
    cfg = SdcConfig(table=table, n_sweeps=config.n_sweeps, preconditioner=config.preconditioner,
                    mode=SweepMode.DIAGONAL_PARALLEL, time_threads=config.n_nodes)
    st = DeviceStepper(problem, cfg, config.dt, serial=False)

    def wall(setup):
        best = math.inf
        for _ in range(max(1, config.reps)):
            setup()
            u = u0.clone()
            st.run(u, 1)
            u.copy_(u0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st.run(u, n)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    rows = []
    for space, tpar in splits + [("device", "fused")]:
        row = {"space_threads": space, "time_threads": tpar,
               "total_threads": space * tpar if isinstance(space, int) else "device",
               "wall_s": float("nan"), "time_per_dof_s": float("nan"), "status": "ok"}
        try:
            if space == "device":
                def setup():
                    st.set_sequential(False)
                    st.set_chains(1)
                    st.set_fused(True)
            elif space != 1:
                raise ConfigError("space_threads has no GPU meaning (the transforms are one device)")
            elif tpar > config.n_nodes:
                raise ConfigError(f"time_threads {tpar} > n_nodes {config.n_nodes}")
            else:
                def setup(tpar=tpar):
                    st.set_fused(False)
                    st.set_sequential(tpar == 1)
                    if tpar > 1:
                        st.set_sequential(False)
                        st.set_chains(tpar)
            w = wall(setup)
            row["wall_s"] = w
            row["time_per_dof_s"] = w / (n * problem.n_dof)
        except (ConfigError, ParameterError) as exc:
            row["status"] = f"skipped: {exc}"
        rows.append(row)
    with open(os.path.join(out_dir, "strong_scaling.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["space_threads", "time_threads", "total_threads", "wall_s",
                                          "time_per_dof_s", "status"])
        w.writeheader()
        w.writerows(rows)
    st.close()
    problem.close()
    return rows


def speedup_report(config, out_dir):
    """Wall-time ratios of each candidate against the configured scheme."""
    os.makedirs(out_dir, exist_ok=True)
    problem = build_problem(config)
    state = build_initial_state(config, problem)
    rows = []
    runs = [(config.scheme, config.dt)] + [(c["scheme"], float(c["dt"])) for c in config.candidates]
    base = None
    for scheme, dt in runs:
        n = config.n_steps(dt)
        best = math.inf
        for _ in range(max(1, config.reps)):
            stepper = build_stepper(config, scheme)
            _, wall = _timed(problem, state, dt, n, stepper)
            if getattr(stepper, "cfg", None) is not None:
                stepper.cfg.close()
            best = min(best, wall)
        base = best if base is None else base
        rows.append({"scheme": scheme, "dt": dt, "n_steps": n, "wall_s": best,
                     "speedup_vs_base": base / best})
    with open(os.path.join(out_dir, "speedup.json"), "w") as f:
        json.dump({"base": config.scheme, "rows": rows}, f, indent=2)
    with open(os.path.join(out_dir, "speedup.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)
    problem.close()
    return rows


def perf_model_report(config, out_dir, n_profile=6):
    """Fit (c_E, c_S) from per-stage CUDA-event timings of sequential-node dSDC
    steps (perfmodel.fit_costs) and compare S_theory with the measured ratio of
    sequential-node to concurrent-node step times on this GPU."""
    import torch

    os.makedirs(out_dir, exist_ok=True)
    problem = build_problem(config)
    state = build_initial_state(config, problem)
    cfg = SdcConfig(table=CollocationTable.radau_right(config.n_nodes), n_sweeps=config.n_sweeps,
                    preconditioner=config.preconditioner, mode=SweepMode.DIAGONAL_PARALLEL,
                    time_threads=config.n_nodes)
    st = DeviceStepper(problem, cfg, config.dt, serial=False)
    u = problem._to_device(state).reshape(-1).contiguous()
    st.set_sequential(True)
    st.profile_step(u)  # warm-up
    reports = [st.profile_step(u) for _ in range(n_profile)]
    model = fit_costs(reports, config.n_nodes)

    def per_step(n=20):
        st.run(u, 2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.run(u, n)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / n

    t_seq = per_step()
    st.set_sequential(False)
    try:  # concurrent node chains (spherical plans; the planar f_E shares one workspace)
        st.set_chains(config.n_nodes)
        t_par_chains = per_step()
        st.set_chains(1)
    except ParameterError:
        t_par_chains = None
    t_par_batched = per_step()
    t_par = min(t for t in (t_par_chains, t_par_batched) if t is not None)
    rep = perf_report(model, s_measured=t_seq / t_par)
    rep.update({"t_step_sequential_s": t_seq, "t_step_parallel_chains_s": t_par_chains,
                "t_step_parallel_batched_s": t_par_batched,
                "stage_reports": [r.__dict__ for r in reports], "environment": environment_info()})
    with open(os.path.join(out_dir, "perf_model.json"), "w") as f:
        json.dump(rep, f, indent=2, default=list)
    st.close()
    problem.close()
    return rep
