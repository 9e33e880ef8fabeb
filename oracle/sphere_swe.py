r"""CPU restatement of the spherical shallow-water split problem.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Parity of the SH
arithmetic is UNPINNED with respect to the reference (it has no spherical
problem, ``SPEC.md:8``); it is pinned by analytic known-answer tests in
``tests/test_oracle_sphere.py`` - including the m > 0 flows of
``tests/sphere_kats.py`` (tilted solid-body rotation, tilted potential flow,
Rossby-Haurwitz wave 4) with a sign-mutation check of every wind-synthesis
term - by the conservation laws of the continuous equations over whole runs
(``tests/sphere_invariants.py``: energy, angular momentum, potential
enstrophy; eight single-term sign mutants fail them) and by the reference
contracts ``pkg/tests/_contracts.py:18-41``.
:class:`SphericalShallowWaterFast` (end of file) is the same problem with the
transforms organised for speed; it is the CPU baseline ``bench.py`` times.

Restated from the planar template ``pkg/src/parsdc/problems/swe.py`` with
``k^2 -> lambda_n = n(n+1)/a^2`` and FFT2 -> spherical-harmonic transform
(SURVEY.md Appendix A):

* ``_f_impl``   <- ``swe.py:157-163``  (-Phibar delta, 0, lambda_n Phi')
* ``_implicit_solve`` <- ``swe.py:165-172`` per-degree 2x2 Helmholtz solve
* ``_f_expl``   <- ``swe.py:174-196``  flux form: Phi'_t = -div(Phi' V),
  zeta_t = -div(eta V), delta_t = curl(eta V) + lambda_n KE
* ``wind_coefs`` <- ``swe.py:200-205`` Helmholtz velocity from psi/chi

Deliberately simple and slow: Legendre sums over *all* nlat latitudes (no
N/S folding, unlike the GPU), ``numpy.fft`` over longitude, tables from
``scipy.special.sph_legendre_p_all`` at Gauss nodes polished in mpmath
(:func:`gauss_nodes`).
"""

import numpy as np
import scipy.special as sps

from paper_2403_20135_b200.core import SplitProblem


_GAUSS = {}


def gauss_nodes(nlat, dps=34):
    """Gauss-Legendre nodes (decreasing) and weights, Newton-polished in mpmath.

    scipy's ``roots_legendre`` weights are only ~1e-10 accurate next to the
    poles at nlat >= 192, so the oracle refines them independently of the
    product (which uses long double): start from scipy's nodes, Newton on
    P_nlat evaluated by its three-term recurrence at ``dps`` digits.
    """
    if nlat in _GAUSS:
        return _GAUSS[nlat]
    from mpmath import mp, mpf

    x0, _ = sps.roots_legendre(nlat)
    half = nlat // 2
    mu = np.empty(nlat)
    w = np.empty(nlat)
    with mp.workdps(dps):
        for i in range(half):
            x = mpf(float(x0[nlat - 1 - i]))
            for it in range(6):
                p0, p1 = mpf(1), x
                for k in range(1, nlat):
                    p0, p1 = p1, ((2 * k + 1) * x * p1 - k * p0) / (k + 1)
                dp = nlat * (x * p1 - p0) / (x * x - 1)
                if it < 5:
                    x = x - p1 / dp
            mu[i] = float(x)
            w[i] = float(2 / ((1 - x * x) * dp * dp))
    mu[half:] = -mu[:half][::-1]
    w[half:] = w[:half][::-1]
    _GAUSS[nlat] = (mu, w)
    return mu, w


def oracle_tables(trunc, nlat):
    """mu (decreasing), w, P[C, nlat], H[C, nlat] from scipy, triangular m-major rows."""
    mu, w = gauss_nodes(nlat)
    theta = np.arccos(mu)
    m_of = np.concatenate([np.full(trunc + 1 - m, m) for m in range(trunc + 1)])
    n_of = np.concatenate([np.arange(m, trunc + 1) for m in range(trunc + 1)])
    p = np.empty((m_of.size, nlat))
    h = np.empty((m_of.size, nlat))
    chunk = max(1, int(2e8 // (16 * (trunc + 1) * (2 * trunc + 1))))
    for j0 in range(0, nlat, chunk):
        th = theta[j0 : j0 + chunk]
        allp = sps.sph_legendre_p_all(trunc, trunc, th, diff_n=1)
        p[:, j0 : j0 + chunk] = allp[0][n_of, m_of]
        h[:, j0 : j0 + chunk] = -np.sin(th)[None, :] * allp[1][n_of, m_of]
    return mu, w, p, h, m_of, n_of


class SphericalShallowWaterOracle(SplitProblem):
    """Spectral-transform rotating shallow water on the sphere, (Phi', zeta, delta) state."""

    def __init__(self, trunc, nlat, nlon, radius=6.371e6, gravity=9.80616, omega=7.292e-5,
                 mean_depth=1.0e4, tables=None):
        super().__init__()
        self.trunc, self.nlat, self.nlon = int(trunc), int(nlat), int(nlon)
        self.radius, self.omega = float(radius), float(omega)
        self.phibar = float(gravity) * float(mean_depth)
        if tables is None:
            tables = oracle_tables(self.trunc, self.nlat)
        self.mu, self.w, self.p, self.h, self.m_of, self.n_of = tables
        self.n_coef = self.m_of.size
        self.state_size = 3 * self.n_coef
        self.lam = self.n_of * (self.n_of + 1.0) / self.radius**2
        self.inv_lam = np.zeros_like(self.lam)
        self.inv_lam[self.n_of > 0] = 1.0 / self.lam[self.n_of > 0]
        self.bounds = np.concatenate([[0], np.cumsum([self.trunc + 1 - m for m in range(self.trunc + 1)])])
        self.coslat2 = 1.0 - self.mu**2

    # -- transforms ----------------------------------------------------------

    def views(self, state):
        c = self.n_coef
        return state[:c], state[c : 2 * c], state[2 * c :]

    def legendre_synthesis(self, coef, tab):
        """F[lat, m] = sum_n coef_nm tab_nm(mu_lat)."""
        out = np.zeros((self.nlat, self.nlon // 2 + 1), dtype=complex)
        for m in range(self.trunc + 1):
            sl = slice(self.bounds[m], self.bounds[m + 1])
            out[:, m] = coef[sl] @ tab[sl]
        return out

    def legendre_analysis(self, fourier, tab, weight):
        """coef_nm = 2 pi sum_lat weight_lat tab_nm(mu_lat) F[lat, m]."""
        out = np.empty(self.n_coef, dtype=complex)
        wf = (2.0 * np.pi * weight)[:, None] * fourier
        for m in range(self.trunc + 1):
            sl = slice(self.bounds[m], self.bounds[m + 1])
            out[sl] = tab[sl] @ wf[:, m]
        return out

    def to_grid(self, fourier):
        return np.fft.irfft(fourier * self.nlon, n=self.nlon, axis=1)

    def to_fourier(self, field):
        return np.fft.rfft(field, axis=1) / self.nlon

    def synthesize(self, coef):
        """Scalar field on the Gaussian grid [nlat, nlon]."""
        return self.to_grid(self.legendre_synthesis(coef, self.p))

    def analyze(self, field):
        return self.legendre_analysis(self.to_fourier(field), self.p, self.w)

    def wind_fourier(self, zeta, delta):
        """Fourier coefficients of U = u cos(phi), V = v cos(phi) (Helmholtz, zero n=0)."""
        a = self.radius
        psi = -zeta * self.inv_lam
        chi = -delta * self.inv_lam
        im = 1j * self.m_of
        uf = (self.legendre_synthesis(im * chi, self.p) - self.legendre_synthesis(psi, self.h)) / a
        vf = (self.legendre_synthesis(im * psi, self.p) + self.legendre_synthesis(chi, self.h)) / a
        return uf, vf

    def div_curl(self, xf, yf, weight):
        """(div, curl) of (X, Y) given as Fourier coefficients, cos-weighted components."""
        im = 1j * self.m_of
        a = self.radius
        wt = weight / self.coslat2
        div = (im * self.legendre_analysis(xf, self.p, wt) - self.legendre_analysis(yf, self.h, wt)) / a
        curl = (im * self.legendre_analysis(yf, self.p, wt) + self.legendre_analysis(xf, self.h, wt)) / a
        return div, curl

    # -- split tendencies ----------------------------------------------------

    def _f_impl(self, state):
        phi, _, delta = self.views(state)
        out = np.empty(self.state_size, dtype=complex)
        c = self.n_coef
        out[:c] = (-self.phibar) * delta
        out[c : 2 * c] = 0.0
        out[2 * c :] = self.lam * phi
        return out

    def solve_coefficients(self, alpha):
        """Host scalars shared bit-for-bit with the GPU kernels."""
        return alpha * self.phibar, alpha * alpha * self.phibar

    def _implicit_solve(self, alpha, beta, guess):
        bphi, bzeta, bdelta = self.views(beta)
        a_phi, a2_phi = self.solve_coefficients(alpha)
        inv = 1.0 / (1.0 + a2_phi * self.lam)
        out = np.empty(self.state_size, dtype=complex)
        c = self.n_coef
        phi = (bphi - a_phi * bdelta) * inv
        out[:c] = phi
        out[c : 2 * c] = bzeta
        out[2 * c :] = bdelta + (alpha * self.lam) * phi
        return out

    def _f_expl(self, state):
        phi, zeta, delta = self.views(state)
        uf, vf = self.wind_fourier(zeta, delta)
        ug, vg = self.to_grid(uf), self.to_grid(vf)
        zg = self.synthesize(zeta)
        pg = self.synthesize(phi)
        eta = zg + (2.0 * self.omega * self.mu)[:, None]
        fa, fb = self.to_fourier(eta * ug), self.to_fourier(eta * vg)
        fc, fd = self.to_fourier(pg * ug), self.to_fourier(pg * vg)
        fke = self.to_fourier((ug * ug + vg * vg) / (2.0 * self.coslat2)[:, None])
        div_mass, _ = self.div_curl(fc, fd, self.w)
        div_abs, curl_abs = self.div_curl(fa, fb, self.w)
        ke = self.legendre_analysis(fke, self.p, self.w)
        out = np.empty(self.state_size, dtype=complex)
        c = self.n_coef
        out[:c] = -div_mass
        out[c : 2 * c] = -div_abs
        out[2 * c :] = curl_abs + self.lam * ke
        real_m0 = self.m_of == 0
        for k in range(3):
            seg = out[k * c : (k + 1) * c]
            seg[real_m0] = seg[real_m0].real
        return out

    # -- diagnostics ---------------------------------------------------------

    def wind(self, state):
        _, zeta, delta = self.views(state)
        uf, vf = self.wind_fourier(zeta, delta)
        cphi = np.sqrt(self.coslat2)[:, None]
        return self.to_grid(uf) / cphi, self.to_grid(vf) / cphi


def relative_l2(a, b, problem):
    """Per-field relative L2 (m>0 weighted x2, Parseval for real fields), SURVEY 8(d)."""
    c = problem.n_coef
    wgt = np.where(problem.m_of > 0, 2.0, 1.0)
    out = []
    for k in range(3):
        x, y = a[k * c : (k + 1) * c], b[k * c : (k + 1) * c]
        num = np.sqrt(np.sum(wgt * np.abs(x - y) ** 2))
        den = np.sqrt(np.sum(wgt * np.abs(y) ** 2))
        out.append(num / den if den > 0 else num)
    return out


class SphericalShallowWaterFast(SphericalShallowWaterOracle):
    """The same problem with the transforms organised the way a CPU spectral
    model runs them (the timed CPU baseline of ``bench.py``; SWEET's SHTns
    backend, ``PAPER.md:171``, is not available here):

    * Legendre synthesis of all fields sharing a table in one matrix product
      per wavenumber (P: zeta, Phi', i m chi, i m psi; H: psi, chi), analysis
      likewise (P: A, B, C, D, KE; H: A, B, D) - 4 table passes per f_E
      instead of 14;
    * N/S folding: only the northern half of each table is read, the southern
      rings follow from parity (P(-mu) = (-1)^(n-m) P(mu), H with the opposite
      sign);
    * stacked FFTs (``scipy.fft`` with ``workers`` threads).

    Same algorithm and operators as :class:`SphericalShallowWaterOracle`; the
    sums are ordered differently, so results agree to rounding (tested at
    1e-13), not bit for bit."""

    def __init__(self, *args, workers=1, **kw):
        super().__init__(*args, **kw)
        self.workers = int(workers)
        half = self.nlat // 2
        # coefficients permuted so that each wavenumber's even (n - m) rows and
        # then its odd rows are contiguous; tables (northern half) in that order
        even = (self.n_of - self.m_of) % 2 == 0
        perm, self.esl, self.osl, pos = [], [], [], 0
        for m in range(self.trunc + 1):
            idx = np.arange(self.bounds[m], self.bounds[m + 1])
            e, o = idx[even[idx]], idx[~even[idx]]
            perm += [e, o]
            self.esl.append(slice(pos, pos + e.size))
            self.osl.append(slice(pos + e.size, pos + e.size + o.size))
            pos += idx.size
        self.perm = np.concatenate(perm)
        self.pp = np.ascontiguousarray(self.p[self.perm, :half])
        self.hp = np.ascontiguousarray(self.h[self.perm, :half])

    def _synth(self, xp, xh):
        """xp [C, kp], xh [C, kh] complex -> Fourier [kp + kh, nlat, nlon/2+1]
        (rows: P fields, then H fields); real matrix products per wavenumber."""
        half = self.nlat // 2
        kp, kh = xp.shape[1], xh.shape[1]
        rp = np.ascontiguousarray(xp[self.perm]).view(np.float64)  # [C, 2 kp] (re, im)
        rh = np.ascontiguousarray(xh[self.perm]).view(np.float64)
        fn = np.zeros((self.trunc + 1, 2, kp + kh, 2, half))  # [m][N/S][field][re/im][lat]
        for m in range(self.trunc + 1):
            e, o = self.esl[m], self.osl[m]
            pe = (rp[e].T @ self.pp[e]).reshape(kp, 2, half)
            po = (rp[o].T @ self.pp[o]).reshape(kp, 2, half)
            he = (rh[e].T @ self.hp[e]).reshape(kh, 2, half)
            ho = (rh[o].T @ self.hp[o]).reshape(kh, 2, half)
            # P: even n-m symmetric about the equator; H: even n-m antisymmetric
            fn[m, 0, :kp], fn[m, 1, :kp] = pe + po, pe - po
            fn[m, 0, kp:], fn[m, 1, kp:] = he + ho, ho - he
        out = np.zeros((kp + kh, self.nlat, self.nlon // 2 + 1), dtype=complex)
        f = fn[..., 0, :] + 1j * fn[..., 1, :]  # [m][N/S][field][lat]
        out[:, :half, : self.trunc + 1] = f[:, 0].transpose(1, 2, 0)
        out[:, half:, : self.trunc + 1] = f[:, 1].transpose(1, 2, 0)[:, ::-1]
        return out

    def _anal(self, gp, gh):
        """Weighted Fourier data gp [kp, nlat, T+1], gh [kh, nlat, T+1] ->
        coefficients [C, kp] (P) and [C, kh] (H)."""
        half = self.nlat // 2

        def fold(g):  # -> symmetric / antisymmetric parts as [m][lat][2 k] real
            s_ = g[:, :half] + g[:, half:][:, ::-1]
            a_ = g[:, :half] - g[:, half:][:, ::-1]
            return (np.ascontiguousarray(s_.transpose(2, 1, 0)).view(np.float64),
                    np.ascontiguousarray(a_.transpose(2, 1, 0)).view(np.float64))

        sp_, ap_ = fold(gp)
        sh_, ah_ = fold(gh)
        cp = np.empty((self.n_coef, 2 * gp.shape[0]))
        ch = np.empty((self.n_coef, 2 * gh.shape[0]))
        for m in range(self.trunc + 1):
            e, o = self.esl[m], self.osl[m]
            cp[e] = self.pp[e] @ sp_[m]
            cp[o] = self.pp[o] @ ap_[m]
            ch[e] = self.hp[e] @ ah_[m]
            ch[o] = self.hp[o] @ sh_[m]
        out_p = np.empty((self.n_coef, gp.shape[0]), dtype=complex)
        out_h = np.empty((self.n_coef, gh.shape[0]), dtype=complex)
        out_p[self.perm] = cp.view(complex)
        out_h[self.perm] = ch.view(complex)
        return out_p, out_h

    def _f_expl(self, state):
        import scipy.fft as sfft

        phi, zeta, delta = self.views(state)
        a = self.radius
        psi, chi = -zeta * self.inv_lam, -delta * self.inv_lam
        im = 1j * self.m_of
        four = self._synth(np.stack([zeta, phi, im * chi, im * psi], axis=1),
                           np.stack([psi, chi], axis=1))
        zf, pf = four[0], four[1]
        uf = (four[2] - four[4]) / a
        vf = (four[3] + four[5]) / a
        g = sfft.irfft(np.stack([uf, vf, zf, pf]) * self.nlon, n=self.nlon, axis=-1, workers=self.workers)
        ug, vg, zg, pg = g
        eta = zg + (2.0 * self.omega * self.mu)[:, None]
        prods = np.stack([eta * ug, eta * vg, pg * ug, pg * vg,
                          (ug * ug + vg * vg) / (2.0 * self.coslat2)[:, None]])
        fa, fb, fc, fd, fke = sfft.rfft(prods, axis=-1, workers=self.workers)[:, :, : self.trunc + 1] / self.nlon
        wc = (2.0 * np.pi * self.w / self.coslat2)[:, None]
        wk = (2.0 * np.pi * self.w)[:, None]
        cp, ch = self._anal(np.stack([fa * wc, fb * wc, fc * wc, fke * wk]),
                            np.stack([fa * wc, fb * wc, fd * wc]))
        div_mass = (im * cp[:, 2] - ch[:, 2]) / a
        div_abs = (im * cp[:, 0] - ch[:, 1]) / a
        curl_abs = (im * cp[:, 1] + ch[:, 0]) / a
        out = np.empty(self.state_size, dtype=complex)
        c = self.n_coef
        out[:c] = -div_mass
        out[c : 2 * c] = -div_abs
        out[2 * c :] = curl_abs + self.lam * cp[:, 3]
        real_m0 = self.m_of == 0
        for k in range(3):
            seg = out[k * c : (k + 1) * c]
            seg[real_m0] = seg[real_m0].real
        return out
