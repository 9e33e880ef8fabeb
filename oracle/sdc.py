"""Restatement of the reference SDC integrators, same floating-point order.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows, function by function:

* ``sweep_init``      <- ``core.initialize_sweep``          core.py:165-174
* ``diag_sweep``      <- ``integrators.diagonal_sweep``      integrators.py:254-288
* ``diag_final``      <- ``integrators._final_node_solve``   integrators.py:291-311
* ``dsdc``            <- ``integrators.dsdc_step``           integrators.py:347-381
* ``serial_pass``     <- ``integrators.serial_sweep``        integrators.py:183-230
* ``serial_sdc``      <- ``integrators.sdc_step_serial``     integrators.py:317-344
* ``march``           <- ``integrators.integrate``           integrators.py:517-554

Every accumulation is written so numpy performs the same roundings in the
same order as the reference (``acc = u0.copy(); acc += w * x`` with ``w`` a
Python float product), which is what lets ``tests/test_oracle_sdc.py`` demand
bit equality with the reference and lets the GPU node kernels be checked
bit-exactly against this file.
"""

import numpy as np

from paper_2403_20135_b200.collocation import DiagonalPreconditioner, diagonal_coefficients
from paper_2403_20135_b200.errors import DivergenceError, NumericalError


class Slots:
    """Per-step storage: step-start triple plus per-node u/fe/fi (core.py:134-162)."""

    def __init__(self, u0, fe0, fi0, m):
        self.u0, self.fe0, self.fi0 = u0, fe0, fi0
        self.u = [u0] * m
        self.fe = [fe0] * m
        self.fi = [fi0] * m


def sweep_init(problem, u_n, m):
    u0 = np.array(u_n, copy=True)
    return Slots(u0, problem.f_expl(u0), problem.f_impl(u0), m)


def _solve(problem, alpha, beta):
    return problem.implicit_solve(alpha, beta, guess=beta)


def diag_rhs(slots, q, dt, diag):
    """Phase one of a diagonal sweep: fold fe += fi, then beta_m into fi[m]."""
    nn = len(slots.fe)
    for j in range(nn):
        slots.fe[j] = slots.fe[j] + slots.fi[j]
    for m in range(nn):
        acc = slots.u0.copy()
        for j in range(nn):
            acc += (dt * q[m, j]) * slots.fe[j]
        acc -= (dt * diag[m]) * slots.fi[m]
        slots.fi[m] = acc


def diag_sweep(problem, slots, table, dt, precond, k, pool=None, threads=1):
    diag = diagonal_coefficients(precond, table, k)
    diag_rhs(slots, table.q_matrix, dt, diag)

    def refresh(nodes):
        for m in nodes:
            u = _solve(problem, dt * diag[m], slots.fi[m])
            slots.fe[m] = problem.f_expl(u)
            slots.fi[m] = problem.f_impl(u)
            slots.u[m] = None

    nn = table.n_nodes
    if pool is None or threads <= 1:
        refresh(range(nn))
    else:
        for fut in [pool.submit(refresh, range(w, nn, threads)) for w in range(threads)]:
            fut.result()


def final_rhs(slots, q, dt, diag):
    last = len(slots.fe) - 1
    acc = slots.u0.copy()
    for j in range(len(slots.fe)):
        w = dt * q[last, j]
        acc += w * slots.fe[j]
        acc += w * slots.fi[j]
    acc -= (dt * diag[last]) * slots.fi[last]
    return acc


def diag_final(problem, slots, table, dt, precond, k):
    diag = diagonal_coefficients(precond, table, k)
    beta = final_rhs(slots, table.q_matrix, dt, diag)
    u = _solve(problem, dt * diag[-1], beta)
    slots.u[-1] = u
    return u


def dsdc(problem, u_n, dt, table, n_sweeps, precond=DiagonalPreconditioner.MIN_SR_FLEX, pool=None,
         threads=1, on_sweep=None):
    slots = sweep_init(problem, u_n, table.n_nodes)
    for k in range(1, n_sweeps):
        diag_sweep(problem, slots, table, dt, precond, k, pool, threads)
        if on_sweep is not None:
            on_sweep(k, slots)
    return diag_final(problem, slots, table, dt, precond, n_sweeps)


def serial_pass(problem, slots, table, dt, forward=True):
    nn = table.n_nodes
    dtau = table.dtau
    ew = np.append(dtau[1:], 0.0) if forward else dtau
    quad = []
    for m in range(nn):
        acc = slots.u0.copy()
        for j in range(nn):
            w = dt * table.q_matrix[m, j]
            acc += w * slots.fe[j]
            acc += w * slots.fi[j]
        quad.append(acc)
    corr = np.zeros_like(slots.u0)
    u = None
    for m in range(nn):
        alpha = dt * dtau[m]
        beta = quad[m]
        beta += corr
        beta -= alpha * slots.fi[m]
        u = _solve(problem, alpha, beta)
        fe_new = problem.f_expl(u)
        fi_new = problem.f_impl(u)
        if m + 1 < nn:
            corr += (dt * ew[m]) * (fe_new - slots.fe[m])
            corr += (dt * dtau[m]) * (fi_new - slots.fi[m])
        slots.fe[m], slots.fi[m], slots.u[m] = fe_new, fi_new, None
    slots.u[-1] = u
    return u


def serial_sdc(problem, u_n, dt, table, n_sweeps, forward=True):
    slots = sweep_init(problem, u_n, table.n_nodes)
    u = None
    for _ in range(n_sweeps):
        u = serial_pass(problem, slots, table, dt, forward)
    return u


def march(problem, u_init, dt, n_steps, step_fn, checkpoint_interval=None, name="dsdc"):
    """Fixed-step driver; returns (times, states) like ``Trajectory`` (integrators.py:517-554)."""
    state = np.array(u_init, copy=True)
    times, states = [0.0], [state.copy()]
    with np.errstate(all="ignore"):
        for step in range(1, n_steps + 1):
            state = step_fn(problem, state, dt)
            if not np.isfinite(state).all():
                comp = int(np.argmin(np.isfinite(state)))
                raise DivergenceError(
                    f"{name} diverged at step {step} of {n_steps}",
                    step_index=step,
                ) from NumericalError("non-finite", component=comp)
            if step == n_steps or (checkpoint_interval and step % checkpoint_interval == 0):
                times.append(step * dt)
                states.append(state.copy())
    return times, states


class DahlquistOracle:
    """u' = lambda_I u + lambda_E u with closed-form solve (ref problems/dahlquist.py:9-53)."""

    def __init__(self, lambda_impl, lambda_expl):
        from paper_2403_20135_b200.core import WorkCounters

        self.lambda_impl = complex(lambda_impl)
        self.lambda_expl = complex(lambda_expl)
        self.counters = WorkCounters()

    def f_expl(self, state):
        self.counters.tally_f_expl()
        return self.lambda_expl * state

    def f_impl(self, state):
        self.counters.tally_f_impl()
        return self.lambda_impl * state

    def implicit_solve(self, alpha, beta, guess=None):
        if alpha == 0.0:
            return beta.copy()
        self.counters.tally_solve()
        return beta / (1.0 - alpha * self.lambda_impl)


# -- reference schemes (integrators.py:387-420) -----------------------------------

THETA = 3.0 / 5.0
W_NOW = 1.5 + 0.1
W_PREV = -(0.5 + 0.1)


def _trap_half(problem, state, dt):
    beta = state + (0.25 * dt) * problem.f_impl(state)
    return problem.implicit_solve(0.25 * dt, beta, guess=beta)


def imex_o2(problem, state, dt):
    u = _trap_half(problem, state, dt)
    rate = problem.f_expl(u)
    pred = u + dt * rate
    u = u + (0.5 * dt) * rate + (0.5 * dt) * problem.f_expl(pred)
    return _trap_half(problem, u, dt)


def theta_step(problem, state, dt, fe_now, fe_prev):
    beta = state + (dt * (1.0 - THETA)) * problem.f_impl(state)
    beta += (dt * W_NOW) * fe_now
    beta += (dt * W_PREV) * fe_prev
    return problem.implicit_solve(THETA * dt, beta, guess=beta)


def ab2_run(problem, state, dt, n_steps):
    """Ab2SiStepper semantics: IMEX-o2 bootstrap, then theta steps with cached history."""
    prev = None
    for _ in range(n_steps):
        now = problem.f_expl(state)
        state = imex_o2(problem, state, dt) if prev is None else theta_step(problem, state, dt, now, prev)
        prev = now
    return state
