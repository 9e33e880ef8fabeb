"""Split-problem contract and evaluation counters (the drop-in boundary).

Same contract as the reference ``SplitProblem`` (``pkg/src/parsdc/core.py:85-126``):
subclasses provide ``_f_expl``, ``_f_impl`` and ``_implicit_solve``; the public
wrappers keep thread-safe evaluation counters exact and ``implicit_solve``
returns an uncounted copy of ``beta`` at ``alpha == 0`` (``core.py:110-114``).
``state_norm`` / ``check_finite`` follow ``core.py:37-50``.

Device-resident problems additionally implement ``tally(n_f_expl, n_f_impl,
n_solve)`` bookkeeping through :meth:`SplitProblem.add_counts`, so a fused GPU
step that evaluates all nodes in one launch still reports the same per-step
counts as the reference's per-node calls.
"""

import threading

import numpy as np

from .errors import NumericalError

__all__ = [
    "SplitProblem",
    "WorkCounters",
    "check_finite",
    "evaluation_counters",
    "state_norm",
]


def state_norm(state):
    """Euclidean norm over the underlying real components (ref ``core.py:37-39``)."""
    return float(np.linalg.norm(state))


def check_finite(state):
    """Raise :class:`NumericalError` naming the first non-finite component (ref ``core.py:42-50``)."""
    finite = np.isfinite(state)
    if not finite.all():
        component = int(np.argmin(finite))
        raise NumericalError(
            f"non-finite value {state.flat[component]!r} at component {component}",
            component=component,
        )


class WorkCounters:
    """Thread-safe tally of tendency evaluations and implicit solves (ref ``core.py:53-82``)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.n_f_expl = 0
        self.n_f_impl = 0
        self.n_solve = 0

    def add(self, n_f_expl=0, n_f_impl=0, n_solve=0):
        with self._lock:
            self.n_f_expl += n_f_expl
            self.n_f_impl += n_f_impl
            self.n_solve += n_solve

    def tally_f_expl(self):
        self.add(n_f_expl=1)

    def tally_f_impl(self):
        self.add(n_f_impl=1)

    def tally_solve(self):
        self.add(n_solve=1)

    def reset(self):
        with self._lock:
            self.n_f_expl = self.n_f_impl = self.n_solve = 0

    def snapshot(self):
        with self._lock:
            return (self.n_f_expl, self.n_f_impl, self.n_solve)


class SplitProblem:
    """Implicit/explicit split right-hand side (ref ``core.py:85-126``).

    ``implicit_solve(alpha, beta)`` returns ``u`` with ``u - alpha f_impl(u) = beta``
    to 1e-12 relative residual and is the identity for ``alpha == 0``.  Every
    evaluation returns a fresh array.
    """

    def __init__(self):
        self.counters = WorkCounters()

    def f_expl(self, state):
        self.counters.tally_f_expl()
        return self._f_expl(state)

    def f_impl(self, state):
        self.counters.tally_f_impl()
        return self._f_impl(state)

    def implicit_solve(self, alpha, beta, guess=None):
        if alpha == 0.0:
            return beta.copy()
        self.counters.tally_solve()
        return self._implicit_solve(alpha, beta, guess)

    def reset_counters(self):
        self.counters.reset()

    def add_counts(self, n_f_expl=0, n_f_impl=0, n_solve=0):
        """Account for evaluations performed inside a fused device launch."""
        self.counters.add(n_f_expl, n_f_impl, n_solve)

    def _f_expl(self, state):
        raise NotImplementedError

    def _f_impl(self, state):
        raise NotImplementedError

    def _implicit_solve(self, alpha, beta, guess):
        raise NotImplementedError


def evaluation_counters(problem):
    """Cumulative ``(n_f_expl, n_f_impl, n_solve)`` (ref ``core.py:129-131``)."""
    return problem.counters.snapshot()
