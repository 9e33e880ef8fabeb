r"""Radau-right collocation constants consumed by the GPU sweep kernels.

Same public surface as the reference (``pkg/src/parsdc/collocation.py:117-256``):
``radau_right_nodes``, ``quadrature_matrix``, ``node_spacings``,
``DiagonalPreconditioner``, ``CollocationTable.radau_right`` and
``diagonal_coefficients``.  The arithmetic is our own: the Radau IIA nodes are
the roots of :math:`P_M(2x-1) - P_{M-1}(2x-1)` (shifted Legendre), found with
``mpmath.polyroots`` at 60 digits and rounded once; the quadrature matrix
integrates the Lagrange basis of the *rounded* node set exactly (60-digit
monomial expansion), as the reference does (``collocation.py:152-196``).  Both
are correct far beyond double precision, so after the final rounding they are
bit-identical to the reference's tables; ``tests/test_collocation.py`` pins
that against golden vectors generated from the reference.
"""

from dataclasses import dataclass
from enum import Enum

import numpy as np
from mpmath import mp

from .errors import ParameterError

MAX_NODES = 16
_DPS = 60


def _shifted_legendre(k):
    """Ascending integer coefficients of P_k(2x - 1)."""
    # P_k(2x-1) = sum_i (-1)^(k+i) C(k,i) C(k+i,i) x^i
    from math import comb

    return [(-1) ** (k + i) * comb(k, i) * comb(k + i, i) for i in range(k + 1)]


def radau_right_nodes(n_nodes):
    """Radau IIA nodes on (0, 1], strictly increasing, last node exactly 1."""
    if not isinstance(n_nodes, (int, np.integer)) or isinstance(n_nodes, bool):
        raise ParameterError(f"node count must be an integer, got {n_nodes!r}")
    if not 1 <= n_nodes <= MAX_NODES:
        raise ParameterError(f"node count must be in [1, {MAX_NODES}], got {n_nodes}")
    if n_nodes == 1:
        return np.array([1.0])
    hi = _shifted_legendre(n_nodes)
    lo = _shifted_legendre(n_nodes - 1) + [0]
    asc = [a - b for a, b in zip(hi, lo)]
    with mp.workdps(_DPS):
        # x = 1 is a root by construction; deflate it exactly, then polish the rest
        desc = [mp.mpf(c) for c in reversed(asc)]
        quot = [desc[0]]
        for c in desc[1:-1]:
            quot.append(c + quot[-1])
        roots = mp.polyroots(quot, maxsteps=400, extraprec=4 * _DPS)
        roots = sorted(mp.re(r) for r in roots)
        poly = lambda x: mp.polyval(desc, x)  # noqa: E731
        dpoly = lambda x: mp.polyval([c * (len(desc) - 1 - i) for i, c in enumerate(desc[:-1])], x)  # noqa: E731
        polished = []
        for r in roots:
            for _ in range(8):
                r = r - poly(r) / dpoly(r)
            polished.append(r)
        nodes = np.array([float(r) for r in polished] + [1.0])
    if np.any(np.diff(nodes) <= 0) or nodes[0] <= 0:
        raise ParameterError(f"root finding failed for M = {n_nodes}")
    return nodes


def quadrature_matrix(nodes):
    """q[m, j] = integral over [0, nodes[m]] of the j-th Lagrange basis polynomial."""
    nodes = np.asarray(nodes, dtype=float)
    if nodes.ndim != 1 or nodes.size == 0:
        raise ParameterError("node set must be a non-empty 1-D array")
    if nodes.size > 1 and np.min(np.diff(nodes)) <= 0.0:
        raise ParameterError("nodes must be strictly increasing")
    m = nodes.size
    q = np.empty((m, m))
    with mp.workdps(_DPS):
        tau = [mp.mpf(float(t)) for t in nodes]
        for j in range(m):
            coef = [mp.mpf(1)]  # ascending monomial coefficients of prod_{i != j}(x - tau_i)
            scale = mp.mpf(1)
            for i in range(m):
                if i != j:
                    coef = [mp.mpf(0)] + coef
                    for p in range(len(coef) - 1):
                        coef[p] -= tau[i] * coef[p + 1]
                    scale *= tau[j] - tau[i]
            anti = [c / (p + 1) for p, c in enumerate(coef)]  # antiderivative / x
            for row in range(m):
                x = tau[row]
                val = mp.mpf(0)
                for c in reversed(anti):
                    val = val * x + c
                q[row, j] = float(val * x / scale)
    return q


def node_spacings(nodes):
    """dtau_1 = tau_1, dtau_m = tau_m - tau_{m-1} (ref ``collocation.py:199-205``)."""
    nodes = np.asarray(nodes, dtype=float)
    dtau = np.diff(nodes, prepend=0.0)
    if np.any(dtau <= 0.0):
        raise ParameterError("nodes must be strictly increasing and positive")
    return dtau


class DiagonalPreconditioner(Enum):
    """Diagonal sweep preconditioners (ref ``collocation.py:208-212``)."""

    MIN_SR_FLEX = "min-sr-flex"
    IMPLICIT_EULER_DTAU = "implicit-euler"


@dataclass(frozen=True)
class CollocationTable:
    """Nodes, quadrature matrix and spacings (ref ``collocation.py:215-230``)."""

    nodes: np.ndarray
    q_matrix: np.ndarray
    dtau: np.ndarray

    @property
    def n_nodes(self):
        return self.nodes.size

    @classmethod
    def radau_right(cls, n_nodes):
        nodes = radau_right_nodes(n_nodes)
        return cls(nodes=nodes, q_matrix=quadrature_matrix(nodes), dtau=node_spacings(nodes))


def diagonal_coefficients(preconditioner, table, sweep_index):
    """q^Delta_{m,m} at one-based sweep k: tau/k (MIN-SR-FLEX) or dtau (ref ``collocation.py:233-256``)."""
    if not isinstance(sweep_index, (int, np.integer)) or sweep_index < 1:
        raise ParameterError(f"sweep index must be a positive integer, got {sweep_index!r}")
    if preconditioner is DiagonalPreconditioner.MIN_SR_FLEX:
        return table.nodes / sweep_index
    if preconditioner is DiagonalPreconditioner.IMPLICIT_EULER_DTAU:
        return table.dtau.copy()
    raise ParameterError(f"unknown preconditioner {preconditioner!r}")
