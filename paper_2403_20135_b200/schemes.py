"""The paper's reference schemes on the GPU.

``imex_o2_step`` / ``ab2_si_step`` and their steppers mirror
``pkg/src/parsdc/integrators.py:387-420, 460-502`` (Strang-split trapezoidal +
Heun IMEX, and the theta = 3/5 two-step semi-implicit scheme) for the
work-precision comparisons of paper Fig. 5.  Every evaluation is a C-ABI call
(f_E, f_I, solve) and every vector update ``x + w * y`` is ``sdcsw_axpy``,
rounded as numpy rounds the reference expression, so the node arithmetic
matches the CPU oracle given the same tendencies.
"""

import time

import numpy as np

from . import _native
from .core import evaluation_counters
from .integrators import StepReport

AB2_THETA = 3.0 / 5.0
AB2_WEIGHT_CURRENT = 1.5 + 0.1
AB2_WEIGHT_PREVIOUS = -(0.5 + 0.1)


class _Dev:
    """Device-state helpers over one problem (states are [1, S] complex128 tensors)."""

    def __init__(self, problem):
        self.p = problem
        self.lib = problem._lib

    def new(self):
        return self.p.empty_states(1)

    def f_expl(self, u):
        return self.p.f_expl_device(u, self.new(), 1)

    def f_impl(self, u):
        return self.p.f_impl_device(u, self.new(), 1)

    def solve(self, alpha, beta):
        if alpha == 0.0:  # identity, not counted (ref core.py:110-114)
            return beta.clone()
        self.p.counters.tally_solve()
        return self.p.implicit_solve_device([alpha], beta, self.new())

    def axpy(self, x, w, y, out=None):
        out = self.new() if out is None else out
        _native.check(self.lib.sdcsw_axpy(2 * x.numel(), x.data_ptr(), float(w), y.data_ptr(),
                                          out.data_ptr(), self.p.stream()), "sdcsw_axpy")
        return out


def _count(problem, fe=0, fi=0):
    problem.counters.add(n_f_expl=fe, n_f_impl=fi)


def _half_step(d, state, dt):
    _count(d.p, fi=1)
    beta = d.axpy(state, 0.25 * dt, d.f_impl(state))
    return d.solve(0.25 * dt, beta)


def imex_o2_device(d, state, dt):
    u = _half_step(d, state, dt)
    _count(d.p, fe=1)
    rate = d.f_expl(u)
    predictor = d.axpy(u, dt, rate)
    _count(d.p, fe=1)
    fe_pred = d.f_expl(predictor)
    u = d.axpy(d.axpy(u, 0.5 * dt, rate), 0.5 * dt, fe_pred)
    return _half_step(d, u, dt)


def theta_device(d, state, dt, fe_now, fe_prev):
    _count(d.p, fi=1)
    beta = d.axpy(state, dt * (1.0 - AB2_THETA), d.f_impl(state))
    beta = d.axpy(beta, dt * AB2_WEIGHT_CURRENT, fe_now, out=beta)
    beta = d.axpy(beta, dt * AB2_WEIGHT_PREVIOUS, fe_prev, out=beta)
    return d.solve(AB2_THETA * dt, beta)


def imex_o2_step(problem, state, dt):
    """One IMEX-o2 step of a device problem; numpy state in and out."""
    d = _Dev(problem)
    out = imex_o2_device(d, problem._to_device(state), dt)
    return out.reshape(-1).cpu().numpy().copy()


class ImexO2Stepper:
    """Adapter running :func:`imex_o2_step` (ref ``integrators.py:460-470``)."""

    name = "imex-o2"

    def reset(self):
        pass

    def step(self, problem, state, dt):
        before = evaluation_counters(problem)
        t0 = time.perf_counter()
        out = imex_o2_step(problem, state, dt)
        d = [a - b for a, b in zip(evaluation_counters(problem), before)]
        return out, StepReport(time.perf_counter() - t0, 0.0, (), 0.0, *d)


class Ab2SiStepper:
    """Two-step semi-implicit scheme, bootstrapped by IMEX-o2 (ref ``integrators.py:473-502``)."""

    name = "ab2-si"

    def __init__(self):
        self._fe_prev = None

    def reset(self):
        self._fe_prev = None

    def step(self, problem, state, dt):
        before = evaluation_counters(problem)
        t0 = time.perf_counter()
        d = _Dev(problem)
        u = problem._to_device(state)
        _count(problem, fe=1)
        fe_now = d.f_expl(u)
        if self._fe_prev is None:
            out = imex_o2_device(d, u, dt)
        else:
            out = theta_device(d, u, dt, fe_now, self._fe_prev)
        self._fe_prev = fe_now
        res = out.reshape(-1).cpu().numpy().copy()
        dd = [a - b for a, b in zip(evaluation_counters(problem), before)]
        return res, StepReport(time.perf_counter() - t0, 0.0, (), 0.0, *dd)


def ab2_si_step(problem, state, state_prev, dt):
    """Single AB2-SI step from (state, state_prev) (ref ``integrators.py:415-420``)."""
    d = _Dev(problem)
    u = problem._to_device(state)
    _count(problem, fe=2)
    out = theta_device(d, u, dt, d.f_expl(u), d.f_expl(problem._to_device(state_prev)))
    return out.reshape(-1).cpu().numpy().copy()


__all__ = ["AB2_THETA", "Ab2SiStepper", "ImexO2Stepper", "ab2_si_step", "imex_o2_step", "np"]
