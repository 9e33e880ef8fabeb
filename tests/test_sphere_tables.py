"""Host-side constants of the product (paper_2403_20135_b200.sphere) against the
independent oracle construction (scipy tables, mpmath Gauss nodes)."""

import numpy as np
import pytest

from oracle.sphere_swe import gauss_nodes, oracle_tables
from paper_2403_20135_b200.sphere import (
    ROW_PAD,
    gaussian_latitudes,
    grid_for,
    laplacian_eigenvalues,
    legendre_tables,
    m_offsets,
    pack_device_tables,
    random_initial_state,
    spectral_index,
    HostTransforms,
)


@pytest.mark.parametrize("nlat", [32, 96, 192])
def test_gauss_latitudes_accuracy(nlat):
    mu, w = gaussian_latitudes(nlat)
    mu2, w2 = gauss_nodes(nlat)
    assert np.max(np.abs(mu - mu2)) < 1e-15
    assert np.max(np.abs(w - w2) / w2) < 2e-15
    assert np.array_equal(mu[: nlat // 2], -mu[::-1][: nlat // 2])


@pytest.mark.parametrize("trunc", [21, 63])
def test_tables_match_scipy(trunc):
    g = grid_for(trunc) if trunc == 63 else None
    nlat = g.nlat if g else 32
    mu, w, p, h, m_of, n_of = oracle_tables(trunc, nlat)
    p2, h2 = legendre_tables(trunc, mu)
    assert np.max(np.abs(p - p2)) < 1e-12
    assert np.max(np.abs(h - h2)) < 1e-11
    mo, no = spectral_index(trunc)
    assert np.array_equal(mo, m_of) and np.array_equal(no, n_of)


def test_layout_and_eigenvalues():
    g = grid_for(63)
    m_of, n_of = spectral_index(63)
    moff = m_offsets(63)
    assert moff[-1] == g.n_coef == (64 * 65) // 2
    for m in (0, 5, 63):
        for n in (m, 63):
            assert m_of[moff[m] + n - m] == m and n_of[moff[m] + n - m] == n
    lam = laplacian_eigenvalues(g)
    assert np.array_equal(lam, n_of * (n_of + 1.0) / g.radius**2)


def test_device_table_packing():
    g = grid_for(63)
    mu, _ = gaussian_latitudes(g.nlat)
    p, h = legendre_tables(63, mu[: g.nlat // 2])
    t = pack_device_tables(g, p, h)
    moff = m_offsets(63)
    for m in range(64):
        r0, r1 = t.rowoff[m], t.rowoff[m + 1]
        le = t.n_even4[m]
        assert le % ROW_PAD == 0 and (r1 - r0 - le) % ROW_PAD == 0
        ns = t.row_n[r0:r1]
        ev, od = ns[:le], ns[le:]
        assert all((n - m) % 2 == 0 for n in ev if n >= 0)
        assert all((n - m) % 2 == 1 for n in od if n >= 0)
        assert sorted(n for n in ns if n >= 0) == list(range(m, 64))
        for r, n in zip(range(r0, r1), ns):
            if n >= 0:
                assert np.array_equal(t.p[r], p[moff[m] + n - m])
            else:
                assert not t.p[r].any() and not t.h[r].any()


def test_initial_state_spec():
    g = grid_for(63)
    u = random_initial_state(g, seed=0)
    c = g.n_coef
    m_of, n_of = spectral_index(63)
    assert np.all(u[:c] == 0)
    assert u[c] == 0 and u[2 * c] == 0
    assert np.all(u[c : 2 * c][m_of == 0].imag == 0)
    tr = HostTransforms(g)
    uu, vv = tr.wind(u[c : 2 * c], u[2 * c :])
    assert abs(np.sqrt(uu * uu + vv * vv).max() - 20.0) < 1e-12
    # delta is 0.1 x the vorticity amplitude: rebuild the draws in the documented order
    rng = np.random.default_rng(0)
    zr, zi, dr, di = (rng.standard_normal(c) for _ in range(4))
    k = n_of > 0
    z_raw = (zr + 1j * zi)[k] * n_of[k] ** -1.5
    d_raw = (dr + 1j * di)[k] * n_of[k] ** -1.5
    z_raw[m_of[k] == 0] = z_raw[m_of[k] == 0].real
    d_raw[m_of[k] == 0] = d_raw[m_of[k] == 0].real
    scale = u[c : 2 * c][k][1] / z_raw[1]
    assert np.allclose(u[c : 2 * c][k], scale * z_raw, rtol=1e-14, atol=0)
    assert np.allclose(u[2 * c :][k], 0.1 * scale * d_raw, rtol=1e-14, atol=0)
    assert np.array_equal(u, random_initial_state(g, seed=0))
