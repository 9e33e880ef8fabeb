"""Snapshot round trip and error behaviour (mirrors pkg/tests/test_problems_swe.py:336-365)."""

import numpy as np
import pytest

from paper_2403_20135_b200.errors import ValidationError
from paper_2403_20135_b200.snapshot import read_snapshot, write_snapshot
from paper_2403_20135_b200.sphere import grid_for, random_initial_state


def test_round_trip(tmp_path):
    g = grid_for(63)
    u = random_initial_state(g, 3)
    write_snapshot(tmp_path / "s.bin", g, u, time=1234.5)
    meta, v = read_snapshot(tmp_path / "s.bin")
    assert np.array_equal(u, v)
    assert meta["time"] == 1234.5 and meta["grid"] == g


def test_errors(tmp_path):
    g = grid_for(63)
    (tmp_path / "bad").write_bytes(b"NOTASNAP" + b"\0" * 100)
    with pytest.raises(ValidationError):
        read_snapshot(tmp_path / "bad")
    write_snapshot(tmp_path / "s.bin", g, random_initial_state(g, 1))
    raw = (tmp_path / "s.bin").read_bytes()
    (tmp_path / "t.bin").write_bytes(raw[:-16])
    with pytest.raises(ValidationError):
        read_snapshot(tmp_path / "t.bin")
    (tmp_path / "h.bin").write_bytes(raw[:20])
    with pytest.raises(ValidationError):
        read_snapshot(tmp_path / "h.bin")
    with pytest.raises(ValidationError):
        write_snapshot(tmp_path / "x.bin", g, np.zeros(5, complex))
