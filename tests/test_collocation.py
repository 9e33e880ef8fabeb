"""Collocation constants: bit-identical to the reference (golden vectors from
parsdc.collocation, tests/golden/make_golden.py) and the reference's own
properties (pkg/tests/test_collocation.py:37-175)."""

import os

import numpy as np
import pytest

from paper_2403_20135_b200.collocation import (
    MAX_NODES,
    CollocationTable,
    DiagonalPreconditioner,
    diagonal_coefficients,
    node_spacings,
    quadrature_matrix,
    radau_right_nodes,
)
from paper_2403_20135_b200.errors import ParameterError

GOLDEN = np.load(os.path.join(os.path.dirname(__file__), "golden", "collocation.npz"))


@pytest.mark.parametrize("m", range(1, MAX_NODES + 1))
def test_tables_bit_identical_to_reference(m):
    t = CollocationTable.radau_right(m)
    assert np.array_equal(t.nodes, GOLDEN[f"nodes_{m}"])
    assert np.array_equal(t.q_matrix, GOLDEN[f"q_{m}"])
    assert np.array_equal(t.dtau, GOLDEN[f"dtau_{m}"])
    for k in (1, 2, 3, 4):
        d = diagonal_coefficients(DiagonalPreconditioner.MIN_SR_FLEX, t, k)
        assert np.array_equal(d, GOLDEN[f"minsr_{m}_{k}"])


def test_radau_known_values():
    assert np.allclose(radau_right_nodes(2), [1.0 / 3.0, 1.0], atol=1e-15)
    s6 = np.sqrt(6.0)
    assert np.allclose(radau_right_nodes(3), [(4 - s6) / 10, (4 + s6) / 10, 1.0], atol=1e-15)


@pytest.mark.parametrize("m", [2, 3, 4, 5, 8])
def test_quadrature_properties(m):
    t = CollocationTable.radau_right(m)
    assert np.allclose(t.q_matrix.sum(axis=1), t.nodes, atol=1e-14)
    for p in range(m):  # exact on polynomials of degree < M
        assert np.allclose(t.q_matrix @ t.nodes**p, t.nodes ** (p + 1) / (p + 1), atol=1e-13)
    assert t.nodes[-1] == 1.0
    assert np.all(np.diff(t.nodes) > 0)


def test_errors():
    with pytest.raises(ParameterError):
        radau_right_nodes(0)
    with pytest.raises(ParameterError):
        radau_right_nodes(MAX_NODES + 1)
    with pytest.raises(ParameterError):
        quadrature_matrix([0.5, 0.2])
    with pytest.raises(ParameterError):
        node_spacings([0.0, 0.5])
    with pytest.raises(ParameterError):
        diagonal_coefficients(DiagonalPreconditioner.MIN_SR_FLEX, CollocationTable.radau_right(2), 0)


def test_live_reference_matches(reference):
    from parsdc import collocation as rc

    for m in (1, 4, 9, 16):
        a, b = CollocationTable.radau_right(m), rc.CollocationTable.radau_right(m)
        assert np.array_equal(a.q_matrix, b.q_matrix) and np.array_equal(a.nodes, b.nodes)
