#!/usr/bin/env python
"""Benchmark: parallel (diagonal) SDC on the spherical shallow-water equations.

Driver contract:

* ``python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config c1]``
* one bench *step* = one full BASELINE run of the configuration (config c1:
  T127 on 384x192, M=4 Radau-right nodes, K=4 sweeps, dt=90 s, 200 time
  steps) from the seeded initial state, state resident in HBM; L2 is flushed
  (256 MiB write) between bench steps and the flush is outside the timed
  events; within a run the Legendre tables stay L2-resident, as in real use.
* ``value`` = simulated time steps per second (whole job), ``e2e`` = the same
  through the public API (``integrate`` with a host numpy state: H2D of the
  initial state and D2H of the final state inside the timed region).
* ``roofline`` = the dominant kernel measured live with CUDA events.
* ``cpu_baseline`` = the CPU oracle (bit-for-bit restatement of the reference
  integrators over the CPU spherical problem) on a bounded sample of steps.
* ``--impl reference`` times that CPU path alone, with every host thread.

Multi-GPU (torchrun, N > 1): nodes are partitioned over ranks (contiguous
blocks), one all-gather of (fe, fi) per sweep over NCCL; the simulation is the
same, so ``scaling`` is "strong".
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c0": dict(trunc=63, nodes=3, sweeps=3, dt=120.0, steps=100, seed=0),
    "c1": dict(trunc=127, nodes=4, sweeps=4, dt=90.0, steps=200, seed=1),
    "c2": dict(trunc=255, nodes=4, sweeps=4, dt=60.0, steps=100, seed=2),
    "c3": dict(trunc=511, nodes=5, sweeps=5, dt=30.0, steps=50, seed=3),
    # ensemble: 64 independent T127 members (seeds 100..163), aggregate member-steps/s;
    # under torchrun the members are sharded over ranks (nodes kept local)
    "c4": dict(trunc=127, nodes=4, sweeps=4, dt=90.0, steps=100, seed=100, members=64),
}
METRIC = "simulated steps/sec (fp64, dSDC)"
UNIT = "steps/s"


def fp64_peak():
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["dmma_tflops"]), d.get("source", "profiles/fp64_peak.json")
    return 37.07, "DMMA microbenchmark tools/probe/dmma_probe.cu on this pool (round 1)"


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json (measured)"
    return 6650.0, "B200_PROFILING.md fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (SM clock, throttle reasons)."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_oracle_rate(cfgname, sample_steps, threads=None):
    """Time the CPU oracle (reference integrator restatement) on a bounded sample."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import sdc as osdc
    from oracle.sphere_swe import SphericalShallowWaterOracle
    from paper_2403_20135_b200 import CollocationTable, random_initial_state
    from paper_2403_20135_b200.sphere import grid_for

    c = CONFIGS[cfgname]
    g = grid_for(c["trunc"])
    prob = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)
    table = CollocationTable.radau_right(c["nodes"])
    u = random_initial_state(g, c["seed"])
    ncpu = os.cpu_count() or 1
    tt = threads if threads is not None else c["nodes"]
    blas = max(1, ncpu // tt)
    try:
        from threadpoolctl import threadpool_limits

        limiter = threadpool_limits(limits=blas)
    except Exception:  # pragma: no cover
        limiter = None
    pool = ThreadPoolExecutor(max_workers=tt) if tt > 1 else None
    try:
        u = osdc.dsdc(prob, u, c["dt"], table, c["sweeps"], pool=pool, threads=tt)  # warm-up
        t0 = time.perf_counter()
        for _ in range(sample_steps):
            u = osdc.dsdc(prob, u, c["dt"], table, c["sweeps"], pool=pool, threads=tt)
        wall = time.perf_counter() - t0
    finally:
        if pool is not None:
            pool.shutdown()
        if limiter is not None:
            limiter.unregister() if hasattr(limiter, "unregister") else None
    cores = min(ncpu, tt * blas)
    return sample_steps / wall, cores, wall


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = CONFIGS[args.config]
    sample = max(1, args.ref_sample)
    rates = []
    cores = 1
    for _ in range(max(0, args.warmup)):
        pass  # the oracle rate function warms itself up once
    for _ in range(max(1, args.steps)):
        r, cores, _ = cpu_oracle_rate(args.config, sample)
        rates.append(r)
    value = float(np.median(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value * c["steps"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded n^-1.5 spectra)",
        "config": {"workload": f"{args.config}: T{c['trunc']} M={c['nodes']} K={c['sweeps']} "
                               f"dt={c['dt']} x{c['steps']} steps", "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{sample} dSDC steps per bench step (of {c['steps']}); "
                                   "reference integrator restated bit-for-bit (oracle/sdc.py), "
                                   "CPU spherical problem oracle/sphere_swe.py, "
                                   f"{c['nodes']} time threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def time_stage(problem, stage, nb, reps=50):
    """Average device duration (s) of one f_E stage launch, CUDA events on its stream."""
    import ctypes

    import torch

    from paper_2403_20135_b200 import _native

    u = problem.empty_states(nb)
    u.zero_()
    out = problem.empty_states(nb)
    lib = problem._lib
    s = problem.stream()
    if stage == 3:  # synthesis alone (as in the step graph): prepare its operand once
        _native.check(lib.sdcsw_transform_stage(problem.handle, 0, u.data_ptr(), out.data_ptr(), nb, s))
    for _ in range(5):
        _native.check(lib.sdcsw_transform_stage(problem.handle, stage, u.data_ptr(), out.data_ptr(), nb, s))
    stream = torch.cuda.current_stream(problem.device)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        lib.sdcsw_transform_stage(problem.handle, stage, u.data_ptr(), out.data_ptr(), nb, s)
    e1.record(stream)
    e1.synchronize()
    del ctypes
    return e0.elapsed_time(e1) * 1e-3 / reps


def stage_roofline(problem, c, members=1, fused=False):
    """Per-stage time per simulated step; roofline of the dominant kernel.

    The sweep launches carry nodes x members states, the init launch members.
    ``fused``: the step runs the analysis with the node-update epilogue
    (transform stage 4), so that is the kernel timed for the analysis."""
    k = c["sweeps"]
    m = c["nodes"] * members
    one = members
    g = problem.grid
    cc, j, ll = g.n_coef, g.nlat // 2, g.trunc + 1
    # algorithmic work per launch for a batch of nb states
    flops = {0: lambda nb: 24.0 * cc * j * nb, 2: lambda nb: 28.0 * cc * j * nb}
    ring_bytes = lambda nb: (8 + 14) * 16.0 * j * ll * nb  # noqa: E731  read Fourier, write analysis data
    per_step = {}
    detail = {}
    for stage, name in ((3, "legendre_synthesis"), (1, "ring_fft_products"),
                        (4 if fused else 2, "legendre_analysis")):
        t1 = time_stage(problem, stage, one)
        tm = time_stage(problem, stage, m)
        per_step[name] = t1 + (k - 1) * tm
        detail[name] = {f"us_nb{one}": t1 * 1e6, f"us_nb{m}": tm * 1e6}
    dom = max(per_step, key=per_step.get)
    tm = detail[dom][f"us_nb{m}"] * 1e-6
    if dom == "ring_fft_products":
        peak, src = hbm_peak()
        ach = ring_bytes(m) / tm / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "peak_source": src}
    else:
        st = 0 if dom == "legendre_synthesis" else 2
        peak, src = fp64_peak()
        ach = flops[st](m) / tm / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "peak_source": src + " (FP64 DMMA)"}
    roof.update({"kernel": dom, "launch_nb": m, "us_per_launch": tm * 1e6, "traffic": None})
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(traffic_path):
        with open(traffic_path) as f:
            tr = json.load(f)
        roof["traffic"] = tr.get(dom)
    return roof, {n: v * 1e6 for n, v in per_step.items()}, detail


def run_device(args):
    import torch

    from paper_2403_20135_b200 import (
        CollocationTable,
        DiagonalSdcStepper,
        SdcConfig,
        SerialSdcStepper,
        SweepMode,
        integrate,
        random_initial_state,
    )
    from paper_2403_20135_b200.integrators import DeviceStepper
    from paper_2403_20135_b200.problem import SphericalShallowWater

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.node_parallel:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29655")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank,
                                world_size=world)
    c = CONFIGS[args.config]
    m_nodes, k_sw, dt, nsteps = c["nodes"], c["sweeps"], c["dt"], c["steps"]
    total_members = c.get("members", 1)
    ensemble = total_members > 1
    if ensemble and total_members % world:
        raise SystemExit(f"{total_members} members do not shard over {world} ranks")
    members = total_members // world if ensemble else 1
    problem = SphericalShallowWater(c["trunc"], device=local, max_batch=max(m_nodes * members, 1))
    if ensemble:
        mem0 = rank * members
        u0_host = np.stack([random_initial_state(problem.grid, c["seed"] + mem0 + e)
                            for e in range(members)])
        u0 = torch.from_numpy(u0_host).to(problem.device).contiguous()
    else:
        u0_host = random_initial_state(problem.grid, c["seed"])
        u0 = problem._to_device(u0_host).reshape(-1).contiguous()
    table = CollocationTable.radau_right(m_nodes)
    cfg = SdcConfig(table=table, n_sweeps=k_sw, mode=SweepMode.DIAGONAL_PARALLEL,
                    time_threads=min(m_nodes, max(1, world)) if world > 1 else 1)
    if world > 1:
        cfg = SdcConfig(table=table, n_sweeps=k_sw, mode=SweepMode.DIAGONAL_PARALLEL,
                        time_threads=min(m_nodes, world))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=problem.device)
    u = torch.empty_like(u0)
    stream = torch.cuda.current_stream(problem.device)

    multi = (world > 1 or args.node_parallel) and not ensemble
    split_plan = False  # the multi-GPU orchestration m-partitioned the plan
    transport = args.transport
    if multi and transport == "p2p":
        # peer mappings must work on every rank, else all ranks take NCCL
        from paper_2403_20135_b200.parallel_nodes import PeerNodeParallelDsdc

        groups = max(g for g in range(1, min(world, m_nodes) + 1) if world % g == 0)
        if c["trunc"] >= 400:
            # table-streaming regime: keep all nodes batched per GEMM (M x the
            # arithmetic intensity) and split the wavenumbers only
            groups = 1
        # collective: peer mappings work on every rank, else every rank takes NCCL
        xpeer, p2p_error = PeerNodeParallelDsdc.create_collective(
            problem, cfg, dt, spectral_parts=world // groups)
        if xpeer is None:
            problem._lib.sdcsw_plan_set_split(problem.handle, 1, 0, None, 0)
            transport = "nccl"
            print(f"[bench] peer exchange unavailable ({p2p_error}); NCCL transport", file=sys.stderr)
    if not multi:
        stepper = DeviceStepper(problem, cfg, dt, serial=False, members=members)
        launches_per_sim_step = stepper.launches_per_step

        def one_run():
            stepper.run(u, nsteps, use_graph=True)
    elif transport == "p2p":
        # node groups x spectral parts (the largest node-group count <= M dividing N);
        # the exchanges run in the kernels over peer memory (analysis epilogue and
        # split synthesis stores + flags), no NCCL on the data path
        split_plan = world // groups > 1
        launches_per_sim_step = xpeer.info()[2]

        def one_run():
            xpeer.run(u, nsteps, use_graph=True)
    else:
        from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend, NodeParallelDsdc

        # node groups x spectral parts: the largest node-group count <= M dividing N
        groups = max(g for g in range(1, min(world, m_nodes) + 1) if world % g == 0)
        spectral = world // groups
        npd = NodeParallelDsdc(CudaNodeBackend(problem), cfg, dt, problem.mean_geopotential,
                               problem.state_size, spectral_parts=spectral)
        split_plan = spectral > 1
        launches_per_sim_step = 3 * (1 + (k_sw - 1)) + (k_sw - 1) + 1
        # the steps (kernels and NCCL all-gathers) replay as CUDA graphs of `chunk` steps
        chunk = max(c for c in range(1, 26) if nsteps % c == 0)
        graph = npd.capture(u, chunk)

        def one_run():
            for _ in range(nsteps // chunk):
                graph.replay()

    def timed_runs(n, timed):
        total = 0.0
        for _ in range(n):
            u.copy_(u0)
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one_run()
            e1.record(stream)
            e1.synchronize()
            total += e0.elapsed_time(e1) * 1e-3
        return total

    timed_runs(args.warmup, False)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t_dev = timed_runs(args.steps, True)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
        t = torch.tensor([t_dev], dtype=torch.float64, device=problem.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_dev = float(t.item())
    sim_steps = args.steps * nsteps
    value = sim_steps * (total_members if ensemble else 1) / t_dev
    node_sweeps = (k_sw - 1) * m_nodes + 1

    # divergence check of the timed runs (device flag)
    finite = bool(torch.isfinite(torch.view_as_real(u)).all().item())

    e2e_multi = None
    if multi:
        # every rank (the graphs hold NCCL collectives): pinned H2D of the initial
        # state, graph replays, D2H of the result; max over ranks
        pinned = torch.from_numpy(u0_host).pin_memory()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            u.copy_(pinned.view_as(u), non_blocking=True)
            one_run()
            out_host = u.cpu()
        t_e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=problem.device)
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        e2e_multi = {"value": sim_steps / float(t_e2e.item()), "unit": UNIT,
                     "h2d_bytes_per_step": int(pinned.numel() * 16),
                     "d2h_bytes_per_step": int(out_host.numel() * 16),
                     "note": "every rank: pinned H2D, node/spectral-parallel graph replays, D2H "
                             "per bench step; max over ranks"}

    result = None
    if rank == 0:
        # --- e2e through the public API (host numpy state in, host state out)
        e2e = None
        if ensemble:
            # public API: host ensemble in (pinned H2D), device run, host ensemble out
            pinned = torch.from_numpy(u0_host).pin_memory()
            ue = torch.empty_like(u0)
            stepper.run(ue.copy_(pinned, non_blocking=True), 1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                ue.copy_(pinned, non_blocking=True)
                stepper.run(ue, nsteps)
                out_host = ue.cpu()
            t_e2e = time.perf_counter() - t0
            e2e = {"value": sim_steps * members / t_e2e, "unit": UNIT,
                   "h2d_bytes_per_step": int(pinned.numel() * 16),
                   "d2h_bytes_per_step": int(out_host.numel() * 16),
                   "note": f"rank 0: {members} members, pinned H2D + DeviceStepper.run + D2H per bench step"}
        elif multi:
            e2e = e2e_multi
        elif world == 1:
            dcfg = SdcConfig(table=table, n_sweeps=k_sw, mode=SweepMode.DIAGONAL_PARALLEL)
            integrate(problem, u0_host, dt, nsteps, DiagonalSdcStepper(dcfg))  # warm-up
            t0 = time.perf_counter()
            for _ in range(args.steps):
                traj = integrate(problem, u0_host, dt, nsteps, DiagonalSdcStepper(dcfg))
            t_e2e = time.perf_counter() - t0
            dcfg.close()
            e2e = {"value": sim_steps / t_e2e, "unit": UNIT,
                   "h2d_bytes_per_step": int(u0_host.nbytes),
                   "d2h_bytes_per_step": int(traj.states[-1].nbytes),
                   "note": f"integrate() with a host numpy state per bench step (one {nsteps}-step run)"}
        # --- serial SDC on one GPU (the paper's sequential baseline)
        scfg = SdcConfig(table=table, n_sweeps=k_sw, mode=SweepMode.SERIAL)
        # serial SDC and the stage timings need an unsplit plan
        aux = (SphericalShallowWater(c["trunc"], device=local, max_batch=max(m_nodes * members, 1))
               if split_plan else problem)
        sst = DeviceStepper(aux, scfg, dt, serial=True)
        us = (u0[0] if ensemble else u0).clone().contiguous()
        sst.run(us, 5)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sst.run(us, nsteps)
        e1.record(stream)
        e1.synchronize()
        serial_rate = nsteps / (e0.elapsed_time(e1) * 1e-3)
        sst.close()
        fused = (not ensemble and world == 1
                 and launches_per_sim_step == 3 * k_sw)  # node updates in the analysis epilogue
        roof, stage_us, stage_detail = stage_roofline(aux, c, members, fused)
        cpu = None
        if world == 1 and not args.no_cpu and not ensemble:
            r, cores, wall = cpu_oracle_rate(args.config, args.cpu_sample)
            cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"{args.cpu_sample} dSDC steps of {args.config} (of {nsteps}) after 1 "
                             f"warm-up step, {wall:.1f} s; oracle/sdc.py (bit-exact restatement of "
                             "the reference integrators) over oracle/sphere_swe.py"}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3,
            "higher_is_better": True,
            "scaling": "weak" if ensemble else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded n^-1.5 SH spectra, max wind 20 m/s)",
            "config": {
                "workload": f"{args.config}: T{c['trunc']} {problem.grid.nlon}x{problem.grid.nlat} "
                            f"M={m_nodes} K={k_sw} dt={dt} s, {nsteps} time steps per bench step"
                            + (f", {total_members} ensemble members ({members} per GPU), value = aggregate member-steps/s"
                               if ensemble else ""),
                "bench_step": f"one full {nsteps}-step run", "l2": "flushed between bench steps (256 MiB write, untimed)",
                "parallelism": ("1 GPU: M nodes as concurrent graph branches / batched GEMM columns" if world == 1 and not multi
                                else f"{world} GPUs: ensemble members sharded" if ensemble
                                else (f"{world} GPUs: node blocks x spectral (m) split; (f_E, f_I) and Fourier parts exchanged over peer memory by the analysis epilogue / split synthesis (no NCCL on the data path)"
                                      if transport == "p2p"
                                      else f"{world} GPUs: node blocks x spectral (m) split, NCCL all-gathers per sweep / per f_E")),
                "ms_per_sim_step": t_dev / sim_steps * 1e3,
                "node_sweeps_per_s": value * node_sweeps,
                "serial_sdc_steps_per_s_1gpu": serial_rate,
                "dsdc_vs_serial_speedup_1gpu": value / serial_rate if (world == 1 and not ensemble) else None,
                "stage_us_per_sim_step": stage_us, "stage_us": stage_detail,
                "finite": finite,
                "multi_gpu_transport": transport if multi else None,
            },
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches_per_sim_step * sim_steps),
            "clocks": clocks.summary(),
        }
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if result is not None:
        print(json.dumps(result), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-sample", type=int, default=4, help="CPU-baseline dSDC steps")
    ap.add_argument("--ref-sample", type=int, default=4, help="reference-arm dSDC steps per bench step")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--node-parallel", action="store_true",
                    help="use the multi-GPU node/spectral orchestration even at world size 1 "
                         "(exercises the N>1 code path on one GPU)")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="multi-GPU exchanges: kernels over peer memory (default) or NCCL all-gathers")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_device(args)


if __name__ == "__main__":
    sys.exit(main())
