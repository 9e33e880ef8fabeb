"""Known-answer tests for the CPU spherical shallow-water oracle:
the SH arithmetic is not in the reference, so it is pinned analytically here."""

import numpy as np
import pytest

from _contracts import assert_implicit_linearity, assert_implicit_solve_contract
from oracle.sphere_swe import SphericalShallowWaterOracle, gauss_nodes, relative_l2
from paper_2403_20135_b200.sphere import SphereGrid, random_initial_state


@pytest.fixture(scope="module")
def small():
    g = SphereGrid(trunc=21, nlat=32, nlon=64)
    return g, SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)


def rand_state(prob, rng, scale=1.0):
    c = prob.n_coef
    x = (rng.standard_normal(3 * c) + 1j * rng.standard_normal(3 * c)) * scale
    for k in range(3):
        seg = x[k * c : (k + 1) * c]
        seg[prob.m_of == 0] = seg[prob.m_of == 0].real
    x[c] = 0.0  # zero-mean vorticity
    x[2 * c] = 0.0  # zero-mean divergence
    return x


def test_gauss_nodes_exactness():
    mu, w = gauss_nodes(32)
    assert abs(w.sum() - 2.0) < 1e-14
    for p in range(0, 63, 2):  # integrates mu^p exactly up to degree 2 nlat - 1
        assert abs(np.sum(w * mu**p) - 2.0 / (p + 1)) < 1e-14
    assert np.all(np.diff(mu) < 0)


def test_synthesis_analysis_round_trip(small):
    g, p = small
    rng = np.random.default_rng(0)
    coef = rand_state(p, rng)[: p.n_coef]
    back = p.analyze(p.synthesize(coef))
    assert np.max(np.abs(back - coef)) < 1e-13 * np.max(np.abs(coef))


# closed-form associated Legendre shapes P(mu) (any normalisation) and dP/dmu
_LEGENDRE_SHAPES = {
    (2, 1): (lambda x: x * np.sqrt(1 - x * x), lambda x: (1 - 2 * x * x) / np.sqrt(1 - x * x)),
    (2, 2): (lambda x: 1 - x * x, lambda x: -2 * x),
    (3, 2): (lambda x: x * (1 - x * x), lambda x: 1 - 3 * x * x),
    (3, 3): (lambda x: (1 - x * x) ** 1.5, lambda x: -3 * x * np.sqrt(1 - x * x)),
    (4, 3): (lambda x: x * (1 - x * x) ** 1.5, lambda x: np.sqrt(1 - x * x) * (1 - 4 * x * x)),
}


@pytest.mark.parametrize("nm", sorted(_LEGENDRE_SHAPES))
def test_laplacian_eigenfunction(small, nm):
    """lap Y_n^m = -n(n+1)/a^2 Y_n^m through synthesis -> grid -> analysis, m > 0.

    For chi = a^2 P(mu) cos(m lam + 0.3) (and the same shape as psi) the wind is
    known in closed form: U = (1/a) d_lam chi, V = ((1 - mu^2)/a) d_mu chi for
    the divergent part, U = -((1 - mu^2)/a) d_mu psi, V = (1/a) d_lam psi for
    the rotational part.  (i) The oracle's spectral wind synthesis (i m P and H
    terms, inverse FFT) reproduces it on the grid; (ii) the divergence / curl
    analysis of the closed-form grid wind returns -n(n+1)/a^2 times the field's
    own coefficients (the Laplacian eigenvalue), and nothing else."""
    g, p = small
    n, m = nm
    pf, dpf = _LEGENDRE_SHAPES[nm]
    a = p.radius
    mu = p.mu[:, None]
    lam = 2 * np.pi * np.arange(p.nlon)[None, :] / p.nlon
    ph = m * lam + 0.3
    field = a * a * pf(mu) * np.cos(ph)
    d_lam = -a * a * m * pf(mu) * np.sin(ph)
    d_mu = a * a * dpf(mu) * np.cos(ph)
    coef = p.analyze(field)
    own = (p.n_of == n) & (p.m_of == m)
    assert np.max(np.abs(coef[~own])) <= 1e-14 * np.max(np.abs(coef))  # one harmonic
    lam_n = n * (n + 1.0) / a**2
    cos2 = 1 - mu * mu
    zero = np.zeros(p.n_coef, complex)
    cases = (  # (zeta, delta) spectral, closed-form (U, V), which of (div, curl) is lap
        (zero, -lam_n * coef, d_lam / a, cos2 * d_mu / a, 0),  # chi = field
        (-lam_n * coef, zero, -cos2 * d_mu / a, d_lam / a, 1),  # psi = field
    )
    for zeta, delta, u_cf, v_cf, which in cases:
        uf, vf = p.wind_fourier(zeta, delta)
        scale = np.max(np.abs(u_cf)) + np.max(np.abs(v_cf))
        assert np.max(np.abs(p.to_grid(uf) - u_cf)) <= 1e-13 * scale
        assert np.max(np.abs(p.to_grid(vf) - v_cf)) <= 1e-13 * scale
        div, curl = p.div_curl(p.to_fourier(u_cf), p.to_fourier(v_cf), p.w)
        lap, other = (div, curl) if which == 0 else (curl, div)
        assert np.linalg.norm(lap - (-lam_n) * coef) <= 1e-12 * lam_n * np.linalg.norm(coef)
        assert np.linalg.norm(other) <= 1e-12 * lam_n * np.linalg.norm(coef)


def test_f_expl_of_rest_is_zero(small):
    g, p = small
    assert np.array_equal(p.f_expl(np.zeros(p.state_size, complex)), np.zeros(p.state_size, complex))


def test_mean_and_reality(small):
    g, p = small
    rng = np.random.default_rng(1)
    u = random_initial_state(g, 3)
    u[: p.n_coef] = 50.0 * rand_state(p, rng)[: p.n_coef]
    fe = p.f_expl(u)
    c = p.n_coef
    assert fe[0] == 0.0  # mass (mean Phi') is conserved exactly
    assert fe[c] == 0.0 and fe[2 * c] == 0.0
    for k in range(3):
        assert np.all(fe[k * c : (k + 1) * c][p.m_of == 0].imag == 0.0)


def test_div_curl_round_trip(small):
    g, p = small
    u = random_initial_state(g, 5)
    c = p.n_coef
    zeta, delta = u[c : 2 * c], u[2 * c :]
    uf, vf = p.wind_fourier(zeta, delta)
    div, curl = p.div_curl(uf, vf, p.w)
    assert np.linalg.norm(curl - zeta) <= 1e-12 * np.linalg.norm(zeta)
    assert np.linalg.norm(div - delta) <= 1e-11 * np.linalg.norm(delta)


def test_solid_body_rotation_is_steady(small):
    """zeta = 2 w mu (solid body, u = w a cos(phi)) with the gradient-wind
    balanced Phi' = -(a^2 Omega w + a^2 w^2 / 2) mu^2 (+const): f_E + f_I = 0."""
    g, p = small
    c = p.n_coef
    w = 1e-6
    mu_field = np.repeat(p.mu[:, None], g.nlon, axis=1)
    x = np.zeros(3 * c, complex)
    x[c : 2 * c] = p.analyze(2.0 * w * mu_field)
    phi = -(p.radius**2 * w * w / 2.0 + p.radius**2 * p.omega * w) * mu_field**2
    x[:c] = p.analyze(phi)
    x[0] = 0.0
    tend = p.f_expl(x) + p.f_impl(x)
    scale = np.linalg.norm(p.f_expl(x))
    assert np.linalg.norm(tend) <= 1e-11 * scale


def test_zonal_flow_has_no_vorticity_tendency(small):
    """A purely zonal (m = 0) flow advects nothing: zeta_t = 0 exactly in exact arithmetic."""
    g, p = small
    c = p.n_coef
    rng = np.random.default_rng(7)
    x = np.zeros(3 * c, complex)
    zonal = p.m_of == 0
    x[c : 2 * c][zonal] = rng.standard_normal(zonal.sum()) * 1e-5
    x[c] = 0.0
    fe = p.f_expl(x)
    assert np.linalg.norm(fe[c : 2 * c]) <= 1e-14 * np.linalg.norm(fe)


def test_contracts(small):
    g, p = small
    rng = np.random.default_rng(2)
    beta = random_initial_state(g, 9)
    beta[: p.n_coef] = 1e3 * rand_state(p, rng)[: p.n_coef]
    assert_implicit_solve_contract(p, beta)
    assert_implicit_linearity(p, rand_state(p, rng), rand_state(p, rng), rng)


def direct_f_expl(p, state):
    """Slow independent f_E: direct (non-FFT) Fourier sums and explicit Legendre
    sums at every grid point, products formed pointwise (SURVEY 8c last KAT)."""
    c = p.n_coef
    lam_ = np.arange(p.nlon) * 2.0 * np.pi / p.nlon
    phi, zeta, delta = state[:c], state[c : 2 * c], state[2 * c :]
    a = p.radius
    psi, chi = -zeta * p.inv_lam, -delta * p.inv_lam
    E = np.exp(1j * np.outer(p.m_of, lam_))  # [C, nlon]
    fac = np.where(p.m_of > 0, 2.0, 1.0)

    def grid(coef, tab):
        # f = sum_nm coef tab e^{i m lambda} + c.c. for m > 0
        vals = (coef[:, None, None] * tab[:, :, None] * E[:, None, :])
        return np.real(np.sum(vals * fac[:, None, None], axis=0))

    im = 1j * p.m_of
    U = (grid(im * chi, p.p) - grid(psi, p.h)) / a
    V = (grid(im * psi, p.p) + grid(chi, p.h)) / a
    Z = grid(zeta, p.p)
    Ph = grid(phi, p.p)
    eta = Z + 2 * p.omega * p.mu[:, None]
    cos2 = (1 - p.mu**2)[:, None]
    A, B, C_, D = eta * U, eta * V, Ph * U, Ph * V
    KE = (U * U + V * V) / (2 * cos2)
    Einv = np.exp(-1j * np.outer(lam_, p.m_of)) / p.nlon  # [nlon, C]

    def ana(field, tab, wt):
        four = field @ Einv  # [nlat, C]
        return 2 * np.pi * np.einsum("jc,cj,j->c", four, tab, wt)

    wt = p.w / (1 - p.mu**2)
    div = lambda X, Y: (im * ana(X, p.p, wt) - ana(Y, p.h, wt)) / a  # noqa: E731
    curl = lambda X, Y: (im * ana(Y, p.p, wt) + ana(X, p.h, wt)) / a  # noqa: E731
    out = np.concatenate([-div(C_, D), -div(A, B), curl(A, B) + p.lam * ana(KE, p.p, p.w)])
    return out


def test_f_expl_vs_direct_sums():
    g = SphereGrid(trunc=10, nlat=16, nlon=32)
    p = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)
    u = random_initial_state(g, 4)
    rng = np.random.default_rng(3)
    u[: p.n_coef] = 100.0 * rand_state(p, rng)[: p.n_coef]
    a, b = p.f_expl(u), direct_f_expl(p, u)
    assert max(relative_l2(a, b, p)) < 1e-12


# ---------------------------------------------------------------------------
# m > 0 known-answer flows (tests/sphere_kats.py derives them): the discrete
# f_E + f_I must equal the analytic tendency to rounding.
# ---------------------------------------------------------------------------
from sphere_kats import field_errors, rossby_haurwitz, tilted_potential, tilted_rotation  # noqa: E402

_KAT_FLOWS = {
    "rotation_a0": lambda o: tilted_rotation(o, 0.0),
    "rotation_a45": lambda o: tilted_rotation(o, np.pi / 4),
    "rotation_a90": lambda o: tilted_rotation(o, np.pi / 2),
    "potential_a45": lambda o: tilted_potential(o, np.pi / 4),
    "potential_a90": lambda o: tilted_potential(o, np.pi / 2),
    "rossby_haurwitz4": rossby_haurwitz,
}


def kat_error(p, name):
    x, want = _KAT_FLOWS[name](p)
    fe, fi = p.f_expl(x), p.f_impl(x)
    err = field_errors(p, fe + fi, want, [fe, fi])
    return max(err[:2]) if name.startswith("rossby") else max(err)  # RH: delta_t not analytic


@pytest.fixture(scope="module")
def t42():
    g = SphereGrid(trunc=42, nlat=64, nlon=128)
    return SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)


@pytest.mark.parametrize("name", sorted(_KAT_FLOWS))
def test_known_answer_flows(small, t42, name):
    for p in (small[1], t42):
        assert kat_error(p, name) <= 1e-10


@pytest.mark.parametrize("flip", ["U_chi_P", "U_psi_H", "V_psi_P", "V_chi_H"])
def test_known_answer_flows_catch_wind_sign_errors(small, flip):
    """Mutation check: flipping the sign of any one term of the wind synthesis
    (U = (i m chi P - psi H)/a, V = (i m psi P + chi H)/a) makes at least one
    known-answer flow fail by O(1)."""
    g, p0 = small
    sign = {k: (-1.0 if k == flip else 1.0) for k in ("U_chi_P", "U_psi_H", "V_psi_P", "V_chi_H")}

    class Mutant(SphericalShallowWaterOracle):
        def wind_fourier(self, zeta, delta):
            a = self.radius
            psi, chi = -zeta * self.inv_lam, -delta * self.inv_lam
            im = 1j * self.m_of
            uf = (sign["U_chi_P"] * self.legendre_synthesis(im * chi, self.p)
                  - sign["U_psi_H"] * self.legendre_synthesis(psi, self.h)) / a
            vf = (sign["V_psi_P"] * self.legendre_synthesis(im * psi, self.p)
                  + sign["V_chi_H"] * self.legendre_synthesis(chi, self.h)) / a
            return uf, vf

    p = Mutant(g.trunc, g.nlat, g.nlon, tables=(p0.mu, p0.w, p0.p, p0.h, p0.m_of, p0.n_of))
    worst = max(kat_error(p, name) for name in _KAT_FLOWS if name != "rotation_a0")
    assert worst > 0.1


# -- H-free formulation (paper_2403_20135_b200/csrc/legendre_ponly.cu) ---------


def _eps(n, m):
    n = np.asarray(n, dtype=float)
    return np.where(n > m, np.sqrt(np.maximum(n * n - m * m, 0.0) / (4.0 * n * n - 1.0)), 0.0)


def _p_extended(o):
    """P_k^m at the oracle's nodes for k = m..T+1 (scipy), one [T+2-m, nlat] block per m."""
    import scipy.special as sps

    t = o.trunc
    allp = sps.sph_legendre_p_all(t + 1, t + 1, np.arccos(o.mu))[0]
    return [allp[m : t + 2, m] for m in range(t + 1)]


@pytest.mark.parametrize("which", ["small", "t42"])
def test_h_recurrence_on_oracle_tables(which, request):
    """H_n = a_n P_{n-1} + b_n P_{n+1}, a_n = (n+1) eps_n, b_n = -n eps_{n+1}: the identity
    the H-free GPU transforms rest on, checked against the oracle's own H table."""
    fx = request.getfixturevalue(which)
    o = fx[1] if isinstance(fx, tuple) else fx
    t = o.trunc
    pext = _p_extended(o)
    for m in range(t + 1):
        sl = slice(o.bounds[m], o.bounds[m + 1])
        n = np.arange(m, t + 1)
        pe = pext[m]  # rows k - m
        lower = np.vstack([np.zeros((1, pe.shape[1])), pe[:-2]])  # P_{n-1}
        rec = ((n + 1) * _eps(n, m))[:, None] * lower - (n * _eps(n + 1, m))[:, None] * pe[1:]
        h = o.h[sl]
        assert np.abs(rec - h).max() <= 1e-13 * max(1.0, np.abs(h).max()), m


@pytest.mark.parametrize("which", ["small", "t42"])
def test_h_free_f_expl_matches_oracle(which, request):
    """numpy restatement of the GPU's H-free chain - operand recurrence (k_xsyn_ponly),
    P-only synthesis to degree T+1, grid products, P analyses of A..E to T+1 and the
    assembly (k_assemble_ponly) - equals the oracle's P/H f_E to rounding."""
    fx = request.getfixturevalue(which)
    o = fx[1] if isinstance(fx, tuple) else fx
    t, a = o.trunc, o.radius
    x = rand_state(o, np.random.default_rng(5), 1e-6)
    phi, zeta, delta = o.views(x)
    psi, chi = -zeta * o.inv_lam, -delta * o.inv_lam
    pext = _p_extended(o)
    nf = o.nlon // 2 + 1
    four = {k: np.zeros((o.nlat, nf), complex) for k in ("u", "v", "z", "p")}
    for m in range(t + 1):
        sl = slice(o.bounds[m], o.bounds[m + 1])
        k = np.arange(m, t + 2)
        ext = lambda v: np.concatenate([v[sl], [0.0]])  # noqa: E731  degree T+1 entry = 0
        ps, cs = ext(psi), ext(chi)
        up1 = lambda v: np.concatenate([v[1:], [0.0]])  # noqa: E731  X_{k+1}
        dn1 = lambda v: np.concatenate([[0.0], v[:-1]])  # noqa: E731  X_{k-1}
        ak1 = (k + 2) * _eps(k + 1, m)  # a_{k+1}
        bk1 = -(k - 1) * _eps(k, m)  # b_{k-1}
        uc = (1j * m * cs - (ak1 * up1(ps) + bk1 * dn1(ps))) / a
        vc = (1j * m * ps + (ak1 * up1(cs) + bk1 * dn1(cs))) / a
        pe = pext[m]
        four["u"][:, m] = uc @ pe
        four["v"][:, m] = vc @ pe
        four["z"][:, m] = ext(zeta) @ pe
        four["p"][:, m] = ext(phi) @ pe
    ug, vg, zg, pg = (o.to_grid(four[k]) for k in ("u", "v", "z", "p"))
    eta = zg + (2.0 * o.omega * o.mu)[:, None]
    prods = [eta * ug, eta * vg, pg * ug, pg * vg, (ug * ug + vg * vg) / (2.0 * o.coslat2)[:, None]]
    fo = [o.to_fourier(f) for f in prods]
    ws = 2.0 * np.pi * o.w / (a * o.coslat2)
    wk = 2.0 * np.pi * o.w
    out = np.empty(o.state_size, complex)
    c = o.n_coef
    for m in range(t + 1):
        sl = slice(o.bounds[m], o.bounds[m + 1])
        n = np.arange(m, t + 1)
        pe = pext[m]
        hat = [pe @ (ws * f[:, m]) for f in fo[:4]] + [pe @ (wk * fo[4][:, m])]
        an, bn = (n + 1) * _eps(n, m), -n * _eps(n + 1, m)
        rec = lambda y: an * np.concatenate([[0.0], y[: len(n) - 1]]) + bn * y[1:]  # noqa: E731
        A, B, C, D, E = hat
        out[sl] = -1j * m * C[:-1] + rec(D)
        out[c + o.bounds[m] : c + o.bounds[m + 1]] = -1j * m * A[:-1] + rec(B)
        out[2 * c + o.bounds[m] : 2 * c + o.bounds[m + 1]] = 1j * m * B[:-1] + rec(A) + o.lam[sl] * E[:-1]
    for k in range(3):
        seg = out[k * c : (k + 1) * c]
        seg[o.m_of == 0] = seg[o.m_of == 0].real
    ref = o.f_expl(x)
    assert max(relative_l2(out, ref, o)) < 1e-12
