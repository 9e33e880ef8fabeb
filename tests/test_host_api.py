"""Host-side API mirrors the reference (integrators.py:86-143 validation,
coefficient expressions of diagonal_sweep / _final_node_solve / serial_sweep)."""

import numpy as np
import pytest

from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode
from paper_2403_20135_b200.collocation import DiagonalPreconditioner, diagonal_coefficients
from paper_2403_20135_b200.errors import ParameterError
from paper_2403_20135_b200.integrators import (
    ExplicitSpacing,
    diagonal_step_coefficients,
    serial_step_coefficients,
)
from paper_2403_20135_b200.parallel_nodes import node_block


def test_config_validation_mirrors_reference():
    t = CollocationTable.radau_right(3)
    assert SdcConfig(table=t).n_sweeps == 3
    with pytest.raises(ParameterError):
        SdcConfig(table=t, n_sweeps=0)
    with pytest.raises(ParameterError):
        SdcConfig(table=t, time_threads=2, mode=SweepMode.DIAGONAL_SEQUENTIAL)
    with pytest.raises(ParameterError):
        SdcConfig(table=t, time_threads=4, mode=SweepMode.DIAGONAL_PARALLEL)
    SdcConfig(table=t, time_threads=3, mode=SweepMode.DIAGONAL_PARALLEL)


def test_live_reference_config_errors(reference):
    from parsdc.integrators import SdcConfig as RC, SweepMode as RM
    from parsdc.collocation import CollocationTable as RT
    from parsdc.errors import ParameterError as RPE

    for kw in (dict(n_sweeps=0), dict(time_threads=2), dict(time_threads=9, mode="par")):
        mode = kw.pop("mode", None)
        with pytest.raises(RPE):
            RC(table=RT.radau_right(3), mode=RM.DIAGONAL_PARALLEL if mode else RM.SERIAL, **kw)
        with pytest.raises(ParameterError):
            SdcConfig(table=CollocationTable.radau_right(3),
                      mode=SweepMode.DIAGONAL_PARALLEL if mode else SweepMode.SERIAL, **kw)


@pytest.mark.parametrize("m,k", [(3, 3), (4, 4), (5, 5), (4, 1)])
def test_diagonal_coefficients_are_reference_expressions(m, k):
    t = CollocationTable.radau_right(m)
    cfg = SdcConfig(table=t, n_sweeps=k, mode=SweepMode.DIAGONAL_SEQUENTIAL)
    dt, phibar = 90.0, 9.80616 * 1e4
    coef = diagonal_step_coefficients(cfg, dt, phibar)
    blk = m * (m + 4)
    assert coef.size == (k - 1) * blk + m + 4
    for s in range(1, k):
        d = diagonal_coefficients(DiagonalPreconditioner.MIN_SR_FLEX, t, s)
        for node in range(m):
            row = coef[(s - 1) * blk + node * (m + 4) : (s - 1) * blk + (node + 1) * (m + 4)]
            assert all(row[j] == dt * t.q_matrix[node, j] for j in range(m))
            a = dt * d[node]
            assert row[m] == a and row[m + 1] == a
            assert row[m + 2] == a * phibar and row[m + 3] == a * a * phibar
    d = diagonal_coefficients(DiagonalPreconditioner.MIN_SR_FLEX, t, k)
    fin = coef[(k - 1) * blk :]
    assert all(fin[j] == dt * t.q_matrix[m - 1, j] for j in range(m))
    assert fin[m] == dt * d[-1]


def test_serial_coefficients():
    t = CollocationTable.radau_right(4)
    for sp in ExplicitSpacing:
        cfg = SdcConfig(table=t, n_sweeps=2, mode=SweepMode.SERIAL, explicit_spacing=sp)
        c = serial_step_coefficients(cfg, 60.0, 1.0)
        ew = np.append(t.dtau[1:], 0.0) if sp is ExplicitSpacing.FORWARD else t.dtau
        assert np.array_equal(c[16:20], np.array([60.0 * x for x in ew]))
        assert np.array_equal(c[20:24], np.array([60.0 * x for x in t.dtau]))


@pytest.mark.parametrize("m,world", [(4, 1), (4, 2), (4, 4), (3, 2), (5, 4), (4, 8)])
def test_node_blocks_partition(m, world):
    seen = []
    for r in range(world):
        lo, cnt, per = node_block(m, world, r)
        assert per == -(-m // world)
        seen.extend(range(lo, lo + cnt))
    assert seen == list(range(m))
