"""Device-resident SDC steppers and driver with the reference's API.

Same public surface as ``pkg/src/parsdc/integrators.py`` for the hot path:
``SweepMode``, ``ExplicitSpacing``, ``SdcConfig`` (``:64-143``), ``StepReport``
(``:146-162``), ``DiagonalSdcStepper`` / ``SerialSdcStepper`` (``:426-457``),
``dsdc_step`` / ``sdc_step_serial`` (``:317-381``), ``Trajectory`` and
``integrate`` (``:505-554``).

With a :class:`~.problem.SphericalShallowWater` the whole step runs on the GPU:
the M node updates of a diagonal sweep - the reference's thread-pool tasks
(``integrators.py:278-288``) - are one batched launch sequence (the node index is
a batch dimension of the transforms), and a step is a replayed CUDA graph.  The
per-node arithmetic (quadrature, diagonal right-hand side, solve) is
bit-identical to the reference given the same tendencies; the host scalars
below are formed with exactly the reference's Python expressions.
"""

import ctypes
import time
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native
from .collocation import CollocationTable, DiagonalPreconditioner, diagonal_coefficients
from .core import check_finite, evaluation_counters
from .errors import DivergenceError, NumericalError, ParameterError

__all__ = [
    "DiagonalSdcStepper",
    "ExplicitSpacing",
    "SdcConfig",
    "SerialSdcStepper",
    "StepReport",
    "SweepMode",
    "Trajectory",
    "dsdc_step",
    "integrate",
    "sdc_step_serial",
    "diagonal_step_coefficients",
    "serial_step_coefficients",
]


class SweepMode(Enum):
    """Node ordering of a sweep (ref ``integrators.py:64-69``)."""

    SERIAL = "serial"
    DIAGONAL_SEQUENTIAL = "diagonal-sequential"
    DIAGONAL_PARALLEL = "diagonal-parallel"


class ExplicitSpacing(Enum):
    """Serial-sweep explicit correction weights (ref ``integrators.py:72-83``)."""

    FORWARD = "forward"
    BACKWARD = "backward"


@dataclass
class SdcConfig:
    """Deferred-correction parameters (ref ``integrators.py:86-143``).

    ``time_threads`` keeps its reference meaning for validation; on the GPU
    the nodes of a diagonal sweep are always processed together (batched), so
    it does not change the arithmetic - exactly the reference's guarantee that
    results are bitwise independent of the thread count.
    """

    table: CollocationTable
    n_sweeps: int = None
    preconditioner: DiagonalPreconditioner = DiagonalPreconditioner.MIN_SR_FLEX
    mode: SweepMode = SweepMode.SERIAL
    time_threads: int = 1
    explicit_spacing: ExplicitSpacing = ExplicitSpacing.FORWARD
    _steppers: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        if self.n_sweeps is None:
            self.n_sweeps = self.table.n_nodes
        if not isinstance(self.n_sweeps, int) or self.n_sweeps < 1:
            raise ParameterError(f"sweep count must be a positive integer, got {self.n_sweeps!r}")
        if not isinstance(self.time_threads, int) or self.time_threads < 1:
            raise ParameterError(f"time_threads must be a positive integer, got {self.time_threads!r}")
        if self.time_threads > 1 and self.mode is not SweepMode.DIAGONAL_PARALLEL:
            raise ParameterError(
                f"time_threads = {self.time_threads} requires mode {SweepMode.DIAGONAL_PARALLEL}, "
                f"got {self.mode}"
            )
        if self.time_threads > self.table.n_nodes:
            raise ParameterError(
                f"time_threads = {self.time_threads} exceeds the {self.table.n_nodes} collocation nodes"
            )

    def close(self):
        for st in self._steppers.values():
            st.close()
        self._steppers.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


@dataclass(frozen=True)
class StepReport:
    """Per-step timing and work accounting (ref ``integrators.py:146-162``)."""

    wall_s: float
    init_s: float
    sweep_s: tuple
    final_node_s: float
    n_f_expl: int
    n_f_impl: int
    n_solve: int


@dataclass
class Trajectory:
    """Checkpointed result of a fixed-step integration (ref ``integrators.py:505-514``)."""

    scheme: str
    dt: float
    n_steps: int
    times: list
    states: list
    reports: list


# -- host scalars (bit-identical to the reference expressions) -------------------


def _solve_scalars(alpha, phibar):
    return alpha * phibar, alpha * alpha * phibar


def _scalars_for(phibar, solve_scalars):
    if solve_scalars is None:
        return lambda alpha: _solve_scalars(alpha, phibar)
    return solve_scalars


def diagonal_step_coefficients(cfg, dt, phibar, solve_scalars=None):
    """Flattened per-sweep node coefficients for the device stepper.

    Sweep k (1..K-1), node m: ``dt * q[m, j]`` for all j (``integrators.py:273-276``),
    ``dt * diag[m]`` (``:276``), then the solve scalars of ``alpha = dt * diag[m]``
    (``:237``).  The final block is row M of the quadrature and
    ``diagonal_coefficients(..., K)`` (``:291-303``).  ``solve_scalars(alpha)``
    gives (alpha Phibar, alpha^2 Phibar) as the problem's own solve forms them
    (default ``alpha * alpha * phibar``).
    """
    scalars = _scalars_for(phibar, solve_scalars)
    table = cfg.table
    m_count = table.n_nodes
    q = table.q_matrix
    out = []
    for k in range(1, cfg.n_sweeps):
        diag = diagonal_coefficients(cfg.preconditioner, table, k)
        for m in range(m_count):
            alpha = dt * diag[m]
            out.extend(dt * q[m, j] for j in range(m_count))
            out.append(dt * diag[m])
            out.append(alpha)
            out.extend(scalars(alpha))
    diag = diagonal_coefficients(cfg.preconditioner, table, cfg.n_sweeps)
    last = m_count - 1
    alpha = dt * diag[last]
    out.extend(dt * q[last, j] for j in range(m_count))
    out.append(dt * diag[last])
    out.append(alpha)
    out.extend(scalars(alpha))
    return np.array(out, dtype=np.float64)


def serial_step_coefficients(cfg, dt, phibar, solve_scalars=None):
    """W = dt*q, dt*explicit weights, dt*dtau, solve scalars (``integrators.py:183-230``)."""
    scalars = _scalars_for(phibar, solve_scalars)
    table = cfg.table
    m_count = table.n_nodes
    dtau = table.dtau
    if cfg.explicit_spacing is ExplicitSpacing.FORWARD:
        ew = np.append(dtau[1:], 0.0)
    else:
        ew = dtau
    out = [dt * table.q_matrix[m, j] for m in range(m_count) for j in range(m_count)]
    out += [dt * ew[m] for m in range(m_count)]
    out += [dt * dtau[m] for m in range(m_count)]
    for m in range(m_count):
        alpha = dt * dtau[m]
        out.append(alpha)
        out.extend(scalars(alpha))
    return np.array(out, dtype=np.float64)


# -- device stepper ----------------------------------------------------------------


class DeviceStepper:
    """One ``sdcsw_stepper``: sweep storage on the GPU plus a CUDA graph of one step."""

    def __init__(self, problem, cfg, dt, serial, members=1):
        self.problem = problem
        self.lib = problem._lib
        self.serial = serial
        self.members = int(members)
        if self.members < 1 or (serial and self.members != 1):
            raise ParameterError("ensembles (members > 1) are supported for diagonal SDC only")
        self.n_nodes = cfg.table.n_nodes
        self.n_sweeps = cfg.n_sweeps
        scalars = getattr(problem, "solve_coefficients", None)
        if serial:
            coef = serial_step_coefficients(cfg, dt, problem.mean_geopotential, scalars)
        else:
            coef = diagonal_step_coefficients(cfg, dt, problem.mean_geopotential, scalars)
        self._coef = np.ascontiguousarray(coef)
        handle = ctypes.c_void_p()
        _native.check(
            self.lib.sdcsw_stepper_create_ensemble(problem.handle, 1 if serial else 0,
                                                   self.n_nodes, self.n_sweeps, self.members,
                                                   _native.dptr(self._coef), self._coef.size,
                                                   ctypes.byref(handle)),
            "sdcsw_stepper_create",
        )
        self.handle = handle
        n = ctypes.c_int()
        _native.check(self.lib.sdcsw_stepper_launches_per_step(handle, ctypes.byref(n)))
        self.launches_per_step = n.value

    def set_chains(self, n):
        """Concurrent node chains per sweep (1 = batched on one stream)."""
        _native.check(self.lib.sdcsw_stepper_set_option(self.handle, 0, int(n)), "set_option")

    def set_sequential(self, on=True):
        """One node update at a time (the DIAGONAL_SEQUENTIAL analogue)."""
        _native.check(self.lib.sdcsw_stepper_set_option(self.handle, 1, int(bool(on))), "set_option")

    def set_fused(self, on=True):
        """Node updates in the analysis epilogue (default where supported: T < 200, M <= 6)."""
        _native.check(self.lib.sdcsw_stepper_set_option(self.handle, 2, int(bool(on))), "set_option")
        n = ctypes.c_int()
        _native.check(self.lib.sdcsw_stepper_launches_per_step(self.handle, ctypes.byref(n)))
        self.launches_per_step = n.value

    def set_graph_steps(self, n):
        """Steps per replayed CUDA graph (1..64; results are bit-identical for any value)."""
        _native.check(self.lib.sdcsw_stepper_set_option(self.handle, 3, int(n)), "set_option")

    def profile_step(self, u):
        """Advance ``u`` one step stage by stage; returns a StepReport with CUDA-event stage times."""
        n = self.n_sweeps + 2
        ms = np.zeros(n)
        _native.check(self.lib.sdcsw_stepper_profile(self.handle, u.data_ptr(), _native.dptr(ms), n,
                                                     self.problem.stream()), "sdcsw_stepper_profile")
        return self._report_from_stages(ms)

    def step_hooked(self, u, on_sweep):
        """Advance ``u`` one step stage by stage, calling ``on_sweep(k, state)``
        after every sweep with a :class:`DeviceSweepState` of the sweep storage
        (``sdcsw_stepper_step_hooked``); returns a StepReport with CUDA-event
        stage times."""
        err = []

        def hook(_user, k):
            try:
                on_sweep(k, DeviceSweepState(self, u, k))
            except BaseException as exc:  # re-raised after the C call returns
                err.append(exc)

        cb = _native.SWEEP_HOOK(hook)
        n = self.n_sweeps + 2
        ms = np.zeros(n)
        _native.check(self.lib.sdcsw_stepper_step_hooked(self.handle, u.data_ptr(), ctypes.cast(cb, ctypes.c_void_p),
                                                         None, _native.dptr(ms), n, self.problem.stream()),
                      "sdcsw_stepper_step_hooked")
        if err:
            raise err[0]
        return self._report_from_stages(ms)

    def _report_from_stages(self, ms):
        self.problem.add_counts(*(c * self.members for c in self.counts_per_step()))
        s = ms * 1e-3
        if self.serial:
            sweeps = tuple(s[1 : 1 + self.n_sweeps])
            return StepReport(float(s[: 1 + self.n_sweeps].sum()), float(s[0]), sweeps, 0.0,
                              *self.counts_per_step())
        sweeps = tuple(s[1 : self.n_sweeps])
        return StepReport(float(s[: self.n_sweeps + 1].sum()), float(s[0]), sweeps,
                          float(s[self.n_sweeps]), *self.counts_per_step())

    def storage(self):
        """(bytes, state-sized buffers) of the stepper's device sweep storage
        (``sdcsw_stepper_storage``)."""
        b, n = ctypes.c_longlong(), ctypes.c_longlong()
        _native.check(self.lib.sdcsw_stepper_storage(self.handle, ctypes.byref(b), ctypes.byref(n)))
        return b.value, n.value

    def counts_per_step(self):
        m, k = self.n_nodes, self.n_sweeps
        if self.serial:
            return 1 + k * m, 1 + k * m, k * m
        n = 1 + (k - 1) * m
        return n, n, (k - 1) * m + 1

    def reset(self):
        _native.check(self.lib.sdcsw_stepper_reset(self.handle, self.problem.stream()))

    def run(self, u, n_steps, use_graph=True):
        """Advance the device state tensor ``u`` (``members`` states) in place."""
        if u.numel() != self.members * self.problem.state_size:
            raise ParameterError("state tensor does not hold `members` states")
        _native.check(
            self.lib.sdcsw_stepper_run(self.handle, u.data_ptr(), int(n_steps), int(bool(use_graph)),
                                       self.problem.stream()),
            "sdcsw_stepper_run",
        )
        self.problem.add_counts(*(c * n_steps * self.members for c in self.counts_per_step()))

    def diverged(self):
        idx = ctypes.c_int()
        _native.check(self.lib.sdcsw_stepper_diverged(self.handle, ctypes.byref(idx)))
        return idx.value

    def close(self):
        if self.handle:
            self.lib.sdcsw_stepper_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceSweepState:
    """What the device step retains after sweep ``k``, shown to ``on_sweep``
    the way the reference's ``SweepState`` is (``core.py:134-162``): ``u0``,
    ``fe0``, ``fi0`` and the node slots ``u``, ``fe``, ``fi`` (one-based node m
    at index m - 1), as numpy arrays copied from the device on access.

    The device step drops the node states once their tendencies are formed
    (the reference drops them too, ``integrators.py:233-246``): ``u`` holds
    ``None``.  ``f_I(u0)`` is not stored either; ``fi0`` recomputes it (not
    counted as an evaluation).  :meth:`distinct_node_arrays` counts the arrays
    the device actually retains between sweeps: u0, fe0 and the M nodes' fe
    and fi, 2M + 2 (the reference's bound is 2M + 3,
    ``pkg/tests/test_integrators.py:228-241``).  Valid inside the callback
    only: the next sweep overwrites the buffers the views copy from."""

    def __init__(self, stepper, u, k):
        self._st, self._u, self.sweep = stepper, u, k
        self.n_nodes = stepper.n_nodes
        fe0, fe, fi = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(stepper.lib.sdcsw_stepper_sweep_state(stepper.handle, int(k), ctypes.byref(fe0),
                                                            ctypes.byref(fe), ctypes.byref(fi)))
        self._ptr = {"fe0": fe0.value, "fe": fe.value, "fi": fi.value}
        self.u = [None] * self.n_nodes

    def _states(self, which, count):
        import torch

        size = self._st.problem.state_size
        ptr = self._ptr[which]

        class _View:
            __cuda_array_interface__ = {"shape": (count, size), "typestr": "<c16", "data": (ptr, False),
                                        "version": 3, "strides": None}

        return torch.as_tensor(_View(), device=self._st.problem.device).cpu().numpy().copy()

    @property
    def u0(self):
        return self._u.reshape(-1).cpu().numpy().copy()

    @property
    def fe0(self):
        return self._states("fe0", 1)[0]

    @property
    def fi0(self):
        p = self._st.problem
        out = p.empty_states(1)
        p.f_impl_device(self._u.reshape(1, -1), out, 1)
        return out[0].cpu().numpy().copy()

    @property
    def fe(self):
        return list(self._states("fe", self.n_nodes))

    @property
    def fi(self):
        return list(self._states("fi", self.n_nodes))

    def distinct_node_arrays(self):
        return 2 + 2 * self.n_nodes


def _is_device_problem(problem):
    return hasattr(problem, "handle") and hasattr(problem, "f_expl_device")


def _device_stepper(cfg, problem, dt, serial):
    key = (id(problem), float(dt), serial)
    st = cfg._steppers.get(key)
    if st is None:
        st = DeviceStepper(problem, cfg, float(dt), serial)
        if not serial and cfg.mode is SweepMode.DIAGONAL_SEQUENTIAL:
            # the reference's sequential mode: one node update after another
            # (bit-identical to the batched parallel mode, as in the reference)
            st.set_sequential(True)
        cfg._steppers[key] = st
    return st


def _one_device_step(problem, u_n, dt, cfg, serial, on_sweep=None):
    import torch

    st = _device_stepper(cfg, problem, dt, serial)
    u = problem._to_device(u_n).reshape(-1).contiguous()
    if on_sweep is not None:  # stage by stage, the callback between sweeps
        report = st.step_hooked(u, on_sweep)
        return u.cpu().numpy().copy(), report
    before = evaluation_counters(problem)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record()
    st.run(u, 1, use_graph=True)
    stop.record()
    stop.synchronize()
    wall = start.elapsed_time(stop) * 1e-3
    after = evaluation_counters(problem)
    d = tuple(a - b for a, b in zip(after, before))
    n_sw = cfg.n_sweeps if serial else cfg.n_sweeps - 1
    report = StepReport(wall_s=wall, init_s=0.0, sweep_s=(0.0,) * n_sw, final_node_s=0.0,
                        n_f_expl=d[0], n_f_impl=d[1], n_solve=d[2])
    return u.cpu().numpy().copy(), report


def dsdc_step(problem, u_n, dt, cfg, on_sweep=None):
    """One diagonal-SDC step on the GPU; returns ``(u, report)`` (ref ``integrators.py:347-381``)."""
    if cfg.mode is SweepMode.SERIAL:
        raise ParameterError(f"diagonal step requires a diagonal mode, got {cfg.mode}")
    return _one_device_step(problem, u_n, dt, cfg, serial=False, on_sweep=on_sweep)


def sdc_step_serial(problem, u_n, dt, cfg, on_sweep=None):
    """One serial-SDC step on the GPU; returns ``(u, report)`` (ref ``integrators.py:317-344``)."""
    if cfg.mode is not SweepMode.SERIAL:
        raise ParameterError(f"serial step requires mode {SweepMode.SERIAL}, got {cfg.mode}")
    return _one_device_step(problem, u_n, dt, cfg, serial=True, on_sweep=on_sweep)


class SerialSdcStepper:
    """Adapter running :func:`sdc_step_serial` (ref ``integrators.py:426-440``)."""

    name = "sdc-serial"
    serial = True

    def __init__(self, cfg):
        if cfg.mode is not SweepMode.SERIAL:
            raise ParameterError(f"serial stepper requires mode {SweepMode.SERIAL}, got {cfg.mode}")
        self.cfg = cfg

    def reset(self):
        pass

    def step(self, problem, state, dt):
        return sdc_step_serial(problem, state, dt, self.cfg)


class DiagonalSdcStepper:
    """Adapter running :func:`dsdc_step` (ref ``integrators.py:443-457``)."""

    name = "dsdc"
    serial = False

    def __init__(self, cfg):
        if cfg.mode is SweepMode.SERIAL:
            raise ParameterError(f"diagonal stepper requires a diagonal mode, got {cfg.mode}")
        self.cfg = cfg

    def reset(self):
        pass

    def step(self, problem, state, dt):
        return dsdc_step(problem, state, dt, self.cfg)


def integrate(problem, initial_state, dt, n_steps, stepper, checkpoint_interval=None,
              stage_timings=False):
    """March ``n_steps`` fixed steps (ref ``integrators.py:517-554``).

    For a device problem and an SDC stepper the state stays in HBM for the
    whole run: steps are replayed CUDA graphs, the per-step finiteness check
    runs on the device, and the host only sees the checkpointed states.  A
    non-finite state raises :class:`DivergenceError` with the same one-based
    step index the reference reports.

    ``stage_timings`` (device path, opt-in): every step runs stage by stage
    with CUDA events (unfused, no graph replay) so each :class:`StepReport`
    carries ``init_s``, ``sweep_s`` and ``final_node_s`` as the reference's do
    - the input of ``perfmodel.fit_costs``.  Results are bit-identical; the
    default graph-replayed path reports the per-step wall time only.
    """
    if dt <= 0.0:
        raise ParameterError(f"step size must be positive, got {dt}")
    if n_steps < 1:
        raise ParameterError(f"step count must be at least 1, got {n_steps}")
    if checkpoint_interval is not None and checkpoint_interval < 1:
        raise ParameterError(f"checkpoint interval must be at least 1, got {checkpoint_interval}")
    stepper.reset()
    state = np.array(initial_state, copy=True)
    check_finite(state)
    times = [0.0]
    states = [state.copy()]
    reports = []
    if not (_is_device_problem(problem) and hasattr(stepper, "cfg")):
        with np.errstate(all="ignore"):
            for step in range(1, n_steps + 1):
                state, report = stepper.step(problem, state, dt)
                reports.append(report)
                try:
                    check_finite(state)
                except NumericalError as exc:
                    raise DivergenceError(
                        f"{stepper.name} diverged at step {step} of {n_steps} (t = {step * dt:g}): {exc}",
                        step_index=step,
                    ) from exc
                if step == n_steps or (checkpoint_interval and step % checkpoint_interval == 0):
                    times.append(step * dt)
                    states.append(state.copy())
        return Trajectory(stepper.name, dt, n_steps, times, states, reports)

    import torch

    st = _device_stepper(stepper.cfg, problem, dt, stepper.serial)
    u = problem._to_device(state).reshape(-1).contiguous()
    st.reset()
    stops = list(range(checkpoint_interval, n_steps, checkpoint_interval)) if checkpoint_interval else []
    stops.append(n_steps)
    done = 0
    per = st.counts_per_step()
    n_sw = stepper.cfg.n_sweeps if stepper.serial else stepper.cfg.n_sweeps - 1
    if stage_timings:
        for step in range(1, n_steps + 1):
            reports.append(st.profile_step(u))
            if step == n_steps or (checkpoint_interval and step % checkpoint_interval == 0):
                bad = st.diverged()
                if bad:
                    raise DivergenceError(
                        f"{stepper.name} diverged at step {bad} of {n_steps} (t = {bad * dt:g})",
                        step_index=bad,
                    ) from NumericalError("non-finite state on device")
                times.append(step * dt)
                states.append(u.cpu().numpy().copy())
        return Trajectory(stepper.name, dt, n_steps, times, states, reports)
    for stop_at in stops:
        seg = stop_at - done
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
        st.run(u, seg, use_graph=True)
        end.record()
        end.synchronize()
        wall = start.elapsed_time(end) * 1e-3 / seg
        bad = st.diverged()
        if bad:
            comp = None
            raise DivergenceError(
                f"{stepper.name} diverged at step {bad} of {n_steps} (t = {bad * dt:g})",
                step_index=bad,
            ) from NumericalError("non-finite state on device", component=comp)
        # one (immutable) report shared by the segment's steps: they replayed as graphs and
        # carry the same averaged wall time
        reports.extend([StepReport(wall, 0.0, (0.0,) * n_sw, 0.0, *per)] * seg)
        done = stop_at
        times.append(done * dt)
        states.append(u.cpu().numpy())  # (a fresh host buffer, owned by the checkpoint)
    return Trajectory(stepper.name, dt, n_steps, times, states, reports)


def wall_clock():
    return time.perf_counter()
