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
* ``roofline`` = the dominant kernel, timed live with CUDA events on the
  states of a running simulation; ``roofline.traffic`` = that kernel's DRAM
  bytes per launch from an ncu capture of the same config and batch
  (``profiles/ncu_traffic_r02.json``), else null.
* ``large_truncation`` = config c3 (T511, M=K=5) in the same run: steps/s and
  the per-kernel stage times with their FP64-DMMA / HBM roofline fractions.
* ``cpu_baseline`` = the CPU port (the reference integrators restated
  bit-for-bit over the CPU spherical problem, batched-field transforms) in
  the reference's three modes - dSDC parallel across nodes, dSDC sequential,
  serial SDC - on the host's physical cores.
* ``--impl reference`` times that CPU path alone (dSDC parallel across nodes,
  every physical core), one simulated time step per bench step.
* ``--plan-only`` prints, per config and N in 2/4/8, the node/spectral
  partition and transport the multi-GPU run would use (no GPU needed).

Multi-GPU (torchrun, N > 1): nodes are partitioned over ranks (contiguous
blocks) with a spectral (m) split inside each node group when N > M; the
exchanges run inside the kernels over peer memory (default) or as NCCL
all-gathers called through the C ABI (``--transport nccl``); the simulation
is the same, so ``scaling`` is "strong".
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
DATA = "synthetic (seeded n^-1.5 SH spectra, max wind 20 m/s)"


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


def physical_cores():
    """Physical cores this process may use (reference harness.py:98-114 records
    psutil.cpu_count(logical=False)); affinity-limited when that is smaller."""
    n = None
    try:
        import psutil

        n = psutil.cpu_count(logical=False)
    except Exception:  # pragma: no cover
        pass
    n = n or os.cpu_count() or 1
    try:
        n = min(n, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        pass
    return max(1, n)


def workload_string(cfgname, nlon, nlat):
    c = CONFIGS[cfgname]
    s = (f"{cfgname}: T{c['trunc']} {nlon}x{nlat} M={c['nodes']} K={c['sweeps']} dt={c['dt']} s, "
         f"{c['steps']} time steps per run")
    if c.get("members", 1) > 1:
        s += f", {c['members']} ensemble members, value = aggregate member-steps/s"
    return s


class CpuPort:
    """The CPU path the reference runs (its integrators, restated bit-for-bit in
    oracle/sdc.py) over the CPU spherical problem (oracle/sphere_swe.py,
    batched-field transforms), in the reference's three modes:
    dsdc_parallel (node updates on a pool of M threads, the paper's OpenMP
    loop), dsdc_sequential and serial_sdc (one node after another, all cores
    to BLAS / FFT)."""

    MODES = ("dsdc_parallel", "dsdc_sequential", "serial_sdc")

    def __init__(self, cfgname, cores=None):
        from oracle import sdc as osdc
        from oracle.sphere_swe import SphericalShallowWaterFast
        from paper_2403_20135_b200 import CollocationTable, random_initial_state
        from paper_2403_20135_b200.sphere import grid_for

        self.osdc = osdc
        self.c = c = CONFIGS[cfgname]
        self.grid = grid_for(c["trunc"])
        self.cores = cores or physical_cores()
        self.m = c["nodes"]
        self.table = CollocationTable.radau_right(self.m)
        self.u0 = random_initial_state(self.grid, c["seed"])
        g = self.grid
        self.prob = SphericalShallowWaterFast(g.trunc, g.nlat, g.nlon, workers=self.cores)

    def threads(self, mode):
        """(time threads, BLAS/FFT threads per time thread)."""
        if mode == "dsdc_parallel":
            tt = min(self.m, self.cores)
            return tt, max(1, self.cores // tt)
        return 1, self.cores

    def stepper(self, mode):
        """A function u -> u advancing one time step in ``mode`` (a context
        manager limits the BLAS threads; the pool lives as long as it)."""
        import contextlib
        from concurrent.futures import ThreadPoolExecutor

        from threadpoolctl import threadpool_limits

        c, osdc = self.c, self.osdc
        tt, blas = self.threads(mode)
        self.prob.workers = blas

        @contextlib.contextmanager
        def ctx():
            pool = ThreadPoolExecutor(max_workers=tt) if tt > 1 else None
            try:
                with threadpool_limits(limits=blas):
                    if mode == "serial_sdc":
                        yield lambda u: osdc.serial_sdc(self.prob, u, c["dt"], self.table, c["sweeps"])
                    else:
                        yield lambda u: osdc.dsdc(self.prob, u, c["dt"], self.table, c["sweeps"],
                                                  pool=pool, threads=tt)
            finally:
                if pool is not None:
                    pool.shutdown()
        return ctx()

    def rate(self, mode, warm=2, reps=3, budget_s=3.5):
        """Steps/s of ``mode``: ``warm`` untimed steps, then the minimum over
        at least ``reps`` timed single steps, repeated until ``budget_s`` seconds
        of timed work (reference bench/harness.py:316, 427-436).  Returns
        (steps/s, timed steps)."""
        with self.stepper(mode) as step:
            u = self.u0
            for _ in range(warm):
                u = step(u)
            best, spent, n = float("inf"), 0.0, 0
            while n < reps or spent < budget_s:
                t0 = time.perf_counter()
                u = step(u)
                dt = time.perf_counter() - t0
                best, spent, n = min(best, dt), spent + dt, n + 1
        return 1.0 / best, n


def cpu_baseline_modes(cfgname):
    """cpu_baseline of the GPU arm: the three reference modes on the host's physical cores."""
    port = CpuPort(cfgname)
    t0 = time.perf_counter()
    timed = {mode: port.rate(mode) for mode in CpuPort.MODES}
    rates = {k: v[0] for k, v in timed.items()}
    wall = time.perf_counter() - t0
    c = CONFIGS[cfgname]
    return {
        "value": rates["dsdc_parallel"], "unit": UNIT, "cores": port.cores, "kind": "port",
        "modes": {k: {"steps_per_s": v, "timed_steps": timed[k][1], "time_threads": port.threads(k)[0],
                      "blas_threads": port.threads(k)[1]} for k, v in rates.items()},
        "dsdc_parallel_vs_serial": rates["dsdc_parallel"] / rates["serial_sdc"],
        "sample": (f"per mode 2 warm-up + min over {min(v[1] for v in timed.values())}-"
                   f"{max(v[1] for v in timed.values())} single {cfgname} steps (of {c['steps']}; 3.5 s of timed steps per mode), "
                   f"{wall:.1f} s total; oracle/sdc.py (bit-exact restatement of the reference "
                   "integrators) over oracle/sphere_swe.py SphericalShallowWaterFast; "
                   f"{port.cores} physical cores"),
    }


def run_reference(args):
    """The reference arm: the CPU port in the reference's dSDC mode (nodes on a
    pool of M threads, BLAS/FFT on the remaining physical cores), one simulated
    time step of the workload per bench step; every number below is timed."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = CONFIGS[args.config]
    port = CpuPort(args.config)
    g = port.grid
    with port.stepper("dsdc_parallel") as step:
        u = port.u0
        for _ in range(max(0, args.warmup)):
            u = step(u)
        times = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            u = step(u)
            times.append(time.perf_counter() - t0)
    total = float(sum(times))
    value = len(times) / total
    tt, blas = port.threads("dsdc_parallel")
    sample = (f"one simulated dSDC time step of {args.config} per bench step ({args.steps} timed after "
              f"{args.warmup} warm-up steps, {total:.2f} s timed; a full run is {c['steps']} steps); "
              "oracle/sdc.py (bit-exact restatement of the reference integrators) over "
              f"oracle/sphere_swe.py SphericalShallowWaterFast; {tt} time threads x {blas} BLAS/FFT threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": total / len(times) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": {"workload": workload_string(args.config, g.nlon, g.nlat),
                   "bench_step": "one simulated time step (bounded CPU sample of the run)",
                   "parallelism": f"cpu: {tt} time threads x {blas} BLAS/FFT threads",
                   "min_ms_per_step": min(times) * 1e3},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": port.cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def hold_device(cycles=4_000_000):
    """Keep the current stream busy (a spin kernel, ~2 ms at 1965 MHz) so the
    host has enqueued every timed launch before the device reaches the start
    event: the events then bracket device time only, not host launch gaps
    (a stage kernel of a few microseconds launched through ctypes, or one
    node kernel right after the L2 flush, would otherwise wait on the host)."""
    import torch

    torch.cuda._sleep(int(cycles))


def time_stage(problem, stage, nb, reps=50):
    """Experiment tools only (tools/): device time (s) of one f_E stage launch on
    zeroed states.  The bench's own numbers come from live_stage_times."""
    import torch

    from paper_2403_20135_b200 import _native

    u = problem.empty_states(nb)
    u.zero_()
    out = problem.empty_states(nb)
    lib = problem._lib
    s = problem.stream()
    if stage == 3:
        _native.check(lib.sdcsw_transform_stage(problem.handle, 0, u.data_ptr(), out.data_ptr(), nb, s))
    for _ in range(5):
        _native.check(lib.sdcsw_transform_stage(problem.handle, stage, u.data_ptr(), out.data_ptr(), nb, s))
    stream = torch.cuda.current_stream(problem.device)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    hold_device()
    e0.record(stream)
    for _ in range(reps):
        lib.sdcsw_transform_stage(problem.handle, stage, u.data_ptr(), out.data_ptr(), nb, s)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


STAGE_NAMES = {3: "legendre_synthesis", 1: "ring_fft_products", 2: "legendre_analysis",
               4: "legendre_analysis"}


def stage_work(problem, name, nb):
    """Algorithmic work of one launch over nb states: (amount, unit, bound).

    Legendre GEMMs with the P and H tables: 24 C J nb flop (synthesis: P on 4
    complex fields, H on 2) and 28 C J nb (analysis: P on 4, H on 3), C =
    (T+1)(T+2)/2, J = nlat/2.  H-free plans
    (problem.uses_ponly, legendre_ponly.cu): P only, to degree T+1 - C' = C + T + 1
    coefficients - 16 C' J nb (4 complex fields) and 20 C' J nb (5); their stage
    times include the operand conversion and the assembly kernels.  Ring kernel: 4
    Fourier fields in and 5 product fields out, 16 B per complex value, nlat (T+1)
    values per field and state."""
    g = problem.grid
    cc, j, ll = g.n_coef, g.nlat // 2, g.trunc + 1
    ponly = getattr(problem, "uses_ponly", False)
    if name == "legendre_synthesis":
        return (16.0 * (cc + ll) if ponly else 24.0 * cc) * j * nb, "flop", "tensor"
    if name == "legendre_analysis":
        return (20.0 * (cc + ll) if ponly else 28.0 * cc) * j * nb, "flop", "tensor"
    return 9.0 * 16.0 * g.nlat * ll * nb, "B", "hbm"


def live_stage_times(problem, states, fused=False, reps=30):
    """Average device time (s) per launch of each f_E stage kernel on the live
    states ``states`` (a running simulation's; nb = len(states)).  The whole
    f_E runs once first so every workspace holds live data; each stage is
    then launched ``reps`` times back to back between CUDA events on its own
    stream.  ``fused``: the analysis timed is the step's fused node-update
    epilogue variant (stage 4; last, since it rewrites the operand)."""
    import torch

    from paper_2403_20135_b200 import _native

    nb = states.shape[0]
    lib, s = problem._lib, problem.stream()
    out = problem.empty_states(nb)
    fi = problem.empty_states(nb)

    def launch(stage):
        dst = fi if stage == 4 else out
        return lib.sdcsw_transform_stage(problem.handle, stage, states.data_ptr(), dst.data_ptr(), nb, s)

    for stage in (0, 1, 2):
        _native.check(launch(stage), "sdcsw_transform_stage")
    if fused:
        problem.f_impl_device(states, fi, nb)
    stream = torch.cuda.current_stream(problem.device)
    times = {}
    for stage in (3, 1, 4 if fused else 2):
        for _ in range(3):
            _native.check(launch(stage), "sdcsw_transform_stage")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        hold_device()
        e0.record(stream)
        for _ in range(reps):
            launch(stage)
        e1.record(stream)
        e1.synchronize()
        times[STAGE_NAMES[stage]] = e0.elapsed_time(e1) * 1e-3 / reps
    return times


def roofline_of(problem, name, nb, seconds, cfgname, fused=False):
    work, unit, bound = stage_work(problem, name, nb)
    if bound == "hbm":
        peak, src = hbm_peak()
        ach = work / seconds / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "peak_source": src, "algorithmic_bytes": work}
    else:
        peak, src = fp64_peak()
        ach = work / seconds / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "peak_source": src + " (FP64 DMMA)", "algorithmic_flop": work}
    tname = name + ("_fused" if fused and name == "legendre_analysis" else "")
    roof.update({"kernel": tname, "launch_nb": nb, "us_per_launch": seconds * 1e6,
                 "traffic": measured_traffic(cfgname, tname, nb)})
    wf = measured_traffic(cfgname, tname, nb, ":smem_wavefronts")
    if bound == "hbm" and wf:
        # the ring kernel's own bound is on chip: its shared-memory traffic (ncu wavefronts of
        # this launch, 128 B each) over the same measured launch time, against 128 B/clk/SM
        ach_s = wf * 128.0 / seconds / 1e9
        roof["smem"] = {"achieved": ach_s, "peak": SMEM_PEAK_GBS, "unit": "GB/s",
                        "frac": ach_s / SMEM_PEAK_GBS, "wavefronts": wf,
                        "peak_source": "1 wavefront (128 B)/clk/SM (ncu's peak) x 148 SMs x 1965 MHz, nominal"}
    if getattr(problem, "uses_ponly", False) and bound == "tensor":
        roof["transforms"] = ("H-free: P to degree T+1 (stage = operand conversion + P synthesis)"
                              if name == "legendre_synthesis" else
                              "H-free: P to degree T+1 (stage = P analysis + recurrence assembly)")
    return roof


def measured_traffic(cfgname, name, nb, what=""):
    """DRAM bytes (read + write) per launch of this kernel at this config and
    batch from an ncu capture (profiles/ncu_traffic_r02.json), or None; what =
    ":smem_wavefronts": its shared-memory wavefronts instead."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        tr = json.load(f)
    return tr.get(cfgname, {}).get(f"{name}:nb{nb}{what}")


# shared-memory bandwidth of the B200: one 128 B wavefront per SM per clock (ncu's peak for
# l1tex__data_pipe_lsu_wavefronts_mem_shared), 148 SMs at the 1965 MHz clock of this pool
# (B200_PROFILING.md); MEASURED_PEAKS.json has no shared-memory figure
SMEM_PEAK_GBS = 148 * 128 * 1.965e9 / 1e9


def live_states(stepper, u, n):
    """n consecutive states of a running simulation (one step apart), starting at u."""
    import torch

    out = [u.clone()]
    x = u.clone()
    for _ in range(n - 1):
        stepper.run(x, 1, use_graph=False)
        out.append(x.clone())
    torch.cuda.synchronize()
    return out


def stage_roofline(problem, c, cfgname, stepper, u, members=1, fused=False):
    """Per-stage time per simulated step (live states) and the roofline of the
    dominant kernel.  Sweep launches carry nodes x members states, the init
    launch members."""
    import torch

    k = c["sweeps"]
    m = c["nodes"] * members
    seq = live_states(stepper, u, c["nodes"])
    one_b = seq[0].reshape(members, -1).contiguous()
    many = torch.cat([x.reshape(members, -1) for x in seq]).contiguous()
    t1 = live_stage_times(problem, one_b)
    tm = live_stage_times(problem, many, fused=fused)
    per_step = {n: t1[n] + (k - 1) * tm[n] for n in tm}
    detail = {n: {f"us_nb{members}": t1[n] * 1e6, f"us_nb{m}": tm[n] * 1e6} for n in tm}
    dom = max(per_step, key=per_step.get)
    roof = roofline_of(problem, dom, m, tm[dom], cfgname, fused)
    return roof, {n: v * 1e6 for n, v in per_step.items()}, detail


def large_truncation_block(cfgname="c3", n_steps=20, warmup=3):
    """Config c3 (T511, M = K = 5) in the same bench run: device-timed steps/s
    (state resident in HBM, CUDA graphs) and every stage kernel of a live step
    against its roofline (Legendre GEMMs: FP64 DMMA; ring, sweep-node and
    final-node kernels: HBM)."""
    import torch

    from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
    from paper_2403_20135_b200.integrators import DeviceStepper, diagonal_step_coefficients
    from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend
    from paper_2403_20135_b200.problem import SphericalShallowWater

    c = CONFIGS[cfgname]
    mm, kk = c["nodes"], c["sweeps"]
    t_setup = time.perf_counter()
    p = SphericalShallowWater(c["trunc"], max_batch=mm)
    cfg = SdcConfig(table=CollocationTable.radau_right(mm), n_sweeps=kk, mode=SweepMode.DIAGONAL_PARALLEL)
    st = DeviceStepper(p, cfg, c["dt"], serial=False)
    u = p._to_device(random_initial_state(p.grid, c["seed"])).reshape(-1).contiguous()
    st.run(u, warmup)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream(p.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    st.run(u, n_steps)
    e1.record(stream)
    e1.synchronize()
    t_steps = e0.elapsed_time(e1) * 1e-3
    rate = n_steps / t_steps
    seq = live_states(st, u, mm)
    many = torch.stack(seq).contiguous()
    t1 = live_stage_times(p, seq[0].reshape(1, -1).contiguous())
    tm = live_stage_times(p, many)
    stages = {}
    for name in tm:
        stages[name] = {"nb1": roofline_of(p, name, 1, t1[name], cfgname),
                        f"nb{mm}": roofline_of(p, name, mm, tm[name], cfgname)}
    # node kernels on live tendencies: the sweep's nodes and the closing solve
    fe, fi = p.empty_states(mm), p.empty_states(mm)
    p.f_expl_device(many, fe, mm)
    p.f_impl_device(many, fi, mm)
    coef = diagonal_step_coefficients(cfg, c["dt"], p.mean_geopotential)
    blk = mm * (mm + 4)
    sc = np.ascontiguousarray(coef[:blk])
    fc = np.ascontiguousarray(coef[(kk - 1) * blk:])
    b = CudaNodeBackend(p)
    sbytes = p.state_size * 16.0

    # node kernels: back-to-back launches cycling over copies of the live operands that
    # together exceed L2 three times over, so every launch streams its inputs from HBM
    # (a single launch after an L2 flush would also time its launch ramp)
    l2_bytes = torch.cuda.get_device_properties(p.device).L2_cache_size
    per_launch = (4 * mm + 1) * sbytes  # sweep: u0, fe, fi in; u, fi out
    nsets = max(2, int(np.ceil(3 * l2_bytes / per_launch)))
    sets = [(seq[0].clone(), fe.clone(), fi.clone(), p.empty_states(mm), p.empty_states(mm),
             p.empty_states(1)) for _ in range(nsets)]

    def timed(fn, reps=4 * nsets):
        for q in range(2 * nsets):
            fn(sets[q % nsets])
        hold_device()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for q in range(reps):
            fn(sets[q % nsets])
        a1.record(stream)
        a1.synchronize()
        return a0.elapsed_time(a1) * 1e-3 / reps

    peak, src = hbm_peak()
    for name, fn, nbytes in (
            ("sweep_nodes", lambda o: b.sweep_nodes(mm, 0, mm, sc, o[0], o[1], 1, o[2], 1, False, o[3], o[4]),
             (1 + 2 * mm) * sbytes + 2 * mm * sbytes),
            ("final_node", lambda o: b.final_node(mm, fc, o[0], o[1], 1, o[2], 1, False, o[5]),
             (2 * mm + 2) * sbytes)):
        t = timed(fn)
        stages[name] = {f"nb{mm}": {"bound": "hbm", "achieved": nbytes / t / 1e9, "peak": peak,
                                     "unit": "GB/s", "frac": nbytes / t / 1e9 / peak, "peak_source": src,
                                     "algorithmic_bytes": nbytes, "kernel": name, "us_per_launch": t * 1e6,
                                     "traffic": measured_traffic(cfgname, name, mm),
                                     "l2": f"cold: {nsets} operand copies ({nsets * per_launch / 2**20:.0f} MiB) "
                                           "cycled by back-to-back launches"}}
    del sets
    per_step_us = {n: (t1[n] + (kk - 1) * tm[n]) * 1e6 for n in tm}
    per_step_us["sweep_nodes"] = (kk - 1) * stages["sweep_nodes"][f"nb{mm}"]["us_per_launch"]
    per_step_us["final_node"] = stages["final_node"][f"nb{mm}"]["us_per_launch"]
    st.close()
    p.close()
    return {
        "workload": workload_string(cfgname, p.grid.nlon, p.grid.nlat),
        "steps_per_s": rate, "ms_per_sim_step": t_steps / n_steps * 1e3,
        "node_sweeps_per_s": rate * ((kk - 1) * mm + 1),
        "timed": f"{n_steps} steps (CUDA graphs, state in HBM) after {warmup} warm-up steps",
        "stages": stages, "stage_us_per_sim_step": per_step_us,
        "setup_s": setup,
        "note": "stage kernels timed on live states of this run (consecutive time steps), "
                "CUDA events on the launching stream; fractions are algorithmic work over the "
                "measured peaks (FP64 DMMA profiles/fp64_peak.json, HBM MEASURED_PEAKS.json)",
    }


def partition_plan(cfgname, world):
    """The multi-GPU layout bench.py uses for ``cfgname`` on ``world`` GPUs (the
    same rules as run_device): ensemble members sharded with nodes local, else
    G node groups (the largest divisor of N that is <= M; G = 1 from T400, so
    every GEMM keeps all nodes batched) x S = N / G spectral parts."""
    from paper_2403_20135_b200.parallel_nodes import node_block, spectral_parts
    from paper_2403_20135_b200.sphere import grid_for

    c = CONFIGS[cfgname]
    g = grid_for(c["trunc"])
    mm = c["nodes"]
    state_bytes = 3 * g.n_coef * 16
    if c.get("members", 1) > 1:
        per = c["members"] // world if c["members"] % world == 0 else None
        return {"layout": "ensemble members sharded, nodes local (replicas, no collective)",
                "members_per_gpu": per, "exchange": None}
    groups = max(q for q in range(1, min(world, mm) + 1) if world % q == 0)
    if c["trunc"] >= 400:
        groups = 1
    parts = world // groups
    owned = spectral_parts(c["trunc"], parts)
    coef_per_part = [int(sum(c_ for m, c_ in enumerate(range(c["trunc"] + 1, 0, -1)) if owned[m] == q))
                     for q in range(parts)]
    blocks = [node_block(mm, groups, q)[:2] for q in range(groups)]
    lp = max(owned.count(q) for q in range(parts))
    own_frac = max(coef_per_part) / g.n_coef
    node_x = 2 * max(b[1] for b in blocks) * state_bytes * own_frac
    four_x = 8 * 16 * (g.nlat // 2) * lp * max(b[1] for b in blocks)
    return {
        "node_groups": groups, "spectral_parts": parts,
        "rank_layout": "rank r -> node group r // S, spectral part r % S",
        "node_blocks": [{"node_lo": lo, "count": n} for lo, n in blocks],
        "wavenumbers_per_part": [owned.count(q) for q in range(parts)],
        "coefficients_per_part": coef_per_part,
        "transport": "peer memory (analysis epilogue / split synthesis stores + device flags); "
                     "NCCL through the C ABI if any rank cannot map its peers",
        "node_exchange_bytes_per_rank_per_sweep": node_x if groups > 1 else 0,
        "fourier_exchange_bytes_per_rank_per_fe": four_x if parts > 1 else 0,
    }


def plan_only():
    out = {"plan_only": True,
           "configs": {name: {str(n): partition_plan(name, n) for n in (2, 4, 8)} for name in CONFIGS}}
    print(json.dumps(out), flush=True)
    return 0


def replica_checksum(u, own=None):
    """Sum of |u| over the entries this rank holds (own: per-field mask, spectral parts)."""
    import torch

    x = u.reshape(-1)
    if own is not None:
        m = torch.from_numpy(np.tile(own, 3)).to(x.device)
        x = x[m]
    return float(torch.sum(torch.abs(x)).item())


def replicas_agree(xpeer, u, dist):
    """Ranks holding the same wavenumbers must hold bitwise-equal states: compare
    checksums of the own entries among the ranks of each spectral part."""
    import torch

    own = xpeer.own_coefficients() if xpeer.nparts > 1 else None
    mine = torch.tensor([float(xpeer.part), replica_checksum(u, own)], dtype=torch.float64,
                        device=u.device)
    every = [torch.zeros_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(every, mine)
    sums = {}
    for t in every:
        sums.setdefault(int(t[0].item()), set()).add(t[1].item())
    return all(len(v) == 1 and np.isfinite(list(v)[0]) for v in sums.values())


def peer_exchange_validated(xpeer, u0, dist):
    """Three steps over the peer exchange with a 5 s wait bound before the timed
    runs; True on every rank iff no wait ran out and the replicas agree."""
    import torch

    from paper_2403_20135_b200.errors import DeviceError

    ok = True
    try:
        xpeer.set_wait_bound(5000)
        v = u0.clone()
        xpeer.run(v, 3, use_graph=False)
        xpeer.diverged()  # DeviceError if a peer did not post within the bound
        ok = replicas_agree(xpeer, v, dist)
        xpeer.reset()
        xpeer.set_wait_bound(30000)
    except DeviceError as exc:
        print(f"[bench] peer exchange validation: {exc}", file=sys.stderr)
        ok = False
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=u0.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return bool(flag.item())


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
        os.environ.setdefault("NCCL_DEBUG", "WARN")  # stdout carries the JSON line only
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
        if xpeer is not None and world > 1 and not peer_exchange_validated(xpeer, u0, dist):
            # first contact of the real multi-process peer path: a wait that ran out or
            # ranks whose replicated states disagree make every rank take NCCL
            xpeer.close()
            xpeer, p2p_error = None, "validation run failed (wait bound or replica mismatch)"
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
    replicas = None
    if multi and world > 1 and transport == "p2p":
        replicas = replicas_agree(xpeer, u, dist)

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
            import gc

            for _ in range(2):  # warm-up (stepper creation, graph capture, host caches)
                integrate(problem, u0_host, dt, nsteps, DiagonalSdcStepper(dcfg))
            gc.collect()
            gc.disable()  # host-timed region: no collector pauses inside it
            run_ms = []
            t0 = time.perf_counter()
            for _ in range(args.steps):
                t1 = time.perf_counter()
                traj = integrate(problem, u0_host, dt, nsteps, DiagonalSdcStepper(dcfg))
                run_ms.append((time.perf_counter() - t1) * 1e3)
            t_e2e = time.perf_counter() - t0
            gc.enable()
            dcfg.close()
            e2e = {"value": sim_steps / t_e2e, "unit": UNIT,
                   "h2d_bytes_per_step": int(u0_host.nbytes),
                   "d2h_bytes_per_step": int(traj.states[-1].nbytes),
                   "run_ms": [round(x, 3) for x in run_ms],
                   "note": f"integrate() with a host numpy state per bench step (one {nsteps}-step run); "
                           "value = all timed runs / their total host time, run_ms lists each"}
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
        # --- stage kernels on live states against their rooflines
        fused = (not ensemble and world == 1
                 and launches_per_sim_step == 3 * k_sw)  # node updates in the analysis epilogue
        dcfg = SdcConfig(table=table, n_sweeps=k_sw, mode=SweepMode.DIAGONAL_PARALLEL)
        rst = DeviceStepper(aux, dcfg, dt, serial=False, members=members)
        live = u.clone() if ensemble else us  # the state of a running simulation (unsplit)
        roof, stage_us, stage_detail = stage_roofline(aux, c, args.config, rst, live, members, fused)
        rst.close()
        large = None
        if world == 1 and not args.no_large:
            large = large_truncation_block("c3")
        cpu = None
        if world == 1 and not args.no_cpu and not ensemble:
            cpu = cpu_baseline_modes(args.config)
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev / args.steps * 1e3,
            "higher_is_better": True,
            "scaling": "weak" if ensemble else "strong",
            "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": {
                "workload": workload_string(args.config, problem.grid.nlon, problem.grid.nlat)
                            + (f" ({members} per GPU)" if ensemble else ""),
                "bench_step": f"one full {nsteps}-step run", "l2": "flushed between bench steps (256 MiB write, untimed)",
                "parallelism": ("1 GPU: M nodes as concurrent graph branches / batched GEMM columns" if world == 1 and not multi
                                else f"{world} GPUs: ensemble members sharded" if ensemble
                                else (f"{world} GPUs: node blocks x spectral (m) split; (f_E, f_I) and Fourier parts exchanged over peer memory by the analysis epilogue / split synthesis (no NCCL on the data path)"
                                      if transport == "p2p"
                                      else f"{world} GPUs: node blocks x spectral (m) split, NCCL all-gathers through the C ABI (sdcsw_allgather_rhs) per sweep / per f_E")),
                "ms_per_sim_step": t_dev / sim_steps * 1e3,
                "node_sweeps_per_s": value * node_sweeps,
                "serial_sdc_steps_per_s_1gpu": serial_rate,
                "dsdc_vs_serial_speedup_1gpu": value / serial_rate if (world == 1 and not ensemble) else None,
                "stage_us_per_sim_step": stage_us, "stage_us": stage_detail,
                "finite": finite,
                "multi_gpu_transport": transport if multi else None,
                "replicas_bitwise_equal": replicas,
            },
            "roofline": roof,
            "large_truncation": large,
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
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    ap.add_argument("--no-large", action="store_true", help="skip the c3 (T511) block")
    ap.add_argument("--plan-only", action="store_true",
                    help="print the multi-GPU partition / transport per config and N (no GPU)")
    ap.add_argument("--node-parallel", action="store_true",
                    help="use the multi-GPU node/spectral orchestration even at world size 1 "
                         "(exercises the N>1 code path on one GPU)")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="multi-GPU exchanges: kernels over peer memory (default) or NCCL all-gathers")
    args = ap.parse_args()
    if args.plan_only:
        return plan_only()
    if args.impl == "reference":
        return run_reference(args)
    return run_device(args)


if __name__ == "__main__":
    sys.exit(main())
