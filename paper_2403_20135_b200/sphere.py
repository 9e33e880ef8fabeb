r"""Spherical-harmonic layout, Gaussian grid, Legendre tables and seeded workloads.

This is the host-side setup of the spherical shallow-water problem that the
reference scopes out (``SPEC.md:8``, ``:270``) and SURVEY.md Appendix A restates.
Nothing here is on the per-step hot path: it builds constants once and uploads
them to the device.

Spectral layout (fixed, documented in DESIGN.md): a state is the flat
complex128 concatenation of three fields ``(Phi', zeta, delta)``, each holding
``C = (T+1)(T+2)/2`` coefficients in triangular m-major order,
``idx(m, n) = m (T+1) - m (m-1)/2 + (n - m)`` for ``0 <= m <= n <= T``.
This mirrors the planar problem's ``(3, ...)`` flat state
(``pkg/src/parsdc/problems/swe.py:127-138``).

Grid: ``nlat`` Gaussian latitudes, ring ``i`` at ``mu_i = sin(phi_i)`` in
*decreasing* order (ring 0 next to the north pole); ring ``i`` and ring
``nlat-1-i`` form the N/S pair ``p = i`` used for parity folding.  ``nlon``
equally spaced longitudes ``lambda_k = 2 pi k / nlon``.

Legendre functions are orthonormal with the Condon-Shortley phase,
``2 pi sum_j w_j P_nm(mu_j) P_n'm(mu_j) = delta_nn'`` (scipy's
``sph_legendre_p`` convention), built here by the standard three-term
recurrence over ``l = n - m`` vectorised over all ``m`` at once; ``H_nm =
(1 - mu^2) dP_nm/dmu = -n mu P_nm + e_nm P_{n-1,m}``.
"""

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError

EARTH_RADIUS = 6.371e6
GRAVITY = 9.80616
OMEGA = 7.292e-5
MEAN_DEPTH = 1.0e4


@dataclass(frozen=True)
class SphereGrid:
    """Truncation, Gaussian grid and physical constants of one problem size."""

    trunc: int
    nlat: int
    nlon: int
    radius: float = EARTH_RADIUS
    gravity: float = GRAVITY
    omega: float = OMEGA
    mean_depth: float = MEAN_DEPTH

    def __post_init__(self):
        t, nlat, nlon = self.trunc, self.nlat, self.nlon
        if not isinstance(t, (int, np.integer)) or t < 1:
            raise ParameterError(f"truncation must be a positive integer, got {t!r}")
        if nlat % 2 or nlat < t + 1:
            raise ParameterError(f"nlat must be even and >= T+1, got {nlat}")
        if nlon < 2 * t + 2:
            raise ParameterError(f"nlon must be >= 2T+2, got {nlon}")
        k = nlon
        while k % 2 == 0:
            k //= 2
        if k not in (1, 3):
            raise ParameterError(f"nlon must be 2^k or 3*2^k, got {nlon}")

    @property
    def mean_geopotential(self):
        return self.gravity * self.mean_depth

    @property
    def n_coef(self):
        return (self.trunc + 1) * (self.trunc + 2) // 2

    @property
    def state_size(self):
        return 3 * self.n_coef

    @property
    def n_dof(self):
        return self.nlat * self.nlon


def grid_for(trunc):
    """The BASELINE grids: T63 192x96, T127 384x192, T255 768x384, T511 1536x768."""
    table = {63: (96, 192), 127: (192, 384), 255: (384, 768), 511: (768, 1536)}
    if trunc in table:
        nlat, nlon = table[trunc]
    else:
        nlon = 3 * (trunc + 1)
        nlat = nlon // 2
    return SphereGrid(trunc=trunc, nlat=nlat, nlon=nlon)


def gaussian_latitudes(nlat):
    """(mu, w) with mu decreasing (north first), Gauss-Legendre on [-1, 1].

    numpy's ``leggauss`` (and scipy's ``roots_legendre``) lose up to 1e-10
    relative accuracy in the weights next to the poles, which the
    ``w / (1 - mu^2)`` analysis weights amplify; here the northern nodes are
    polished by Newton steps on the three-term recurrence in long double, the
    weights are ``2 / ((1 - x^2) P_N'(x)^2)`` in long double, and the southern
    half is the exact mirror image.
    """
    x0, _ = np.polynomial.legendre.leggauss(nlat)
    x = np.array(x0[::-1][: nlat // 2], dtype=np.longdouble)
    one = np.longdouble(1)
    for _ in range(4):
        p0, p1 = np.ones_like(x), x.copy()
        for k in range(1, nlat):
            p0, p1 = p1, ((2 * k + 1) * x * p1 - k * p0) / (k + 1)
        dp = nlat * (x * p1 - p0) / (x * x - one)
        x = x - p1 / dp
    p0, p1 = np.ones_like(x), x.copy()
    for k in range(1, nlat):
        p0, p1 = p1, ((2 * k + 1) * x * p1 - k * p0) / (k + 1)
    dp = nlat * (x * p1 - p0) / (x * x - one)
    w = 2 / ((one - x * x) * dp * dp)
    xn = x.astype(np.float64)
    wn = w.astype(np.float64)
    return np.concatenate([xn, -xn[::-1]]), np.concatenate([wn, wn[::-1]])


def spectral_index(trunc):
    """Arrays (m_of, n_of) of length C in the triangular m-major layout."""
    ms, ns = [], []
    for m in range(trunc + 1):
        ms.append(np.full(trunc + 1 - m, m))
        ns.append(np.arange(m, trunc + 1))
    return np.concatenate(ms), np.concatenate(ns)


def m_offsets(trunc):
    m = np.arange(trunc + 2)
    return m * (trunc + 1) - m * (m - 1) // 2


def laplacian_eigenvalues(grid):
    """lambda_n = n (n+1) / a^2 per coefficient (the sphere's k^2)."""
    _, n = spectral_index(grid.trunc)
    return n * (n + 1.0) / grid.radius**2


def legendre_tables(trunc, mu):
    """P[idx, j] and H[idx, j] for every coefficient idx and latitude mu_j.

    Recurrence (vectorised over m for each l = n - m):
    P_mm = (-1)^m sqrt((2m+1)/(4 pi) prod_{k<=m} (2k-1)/(2k)) sin^m theta,
    P_{m+1,m} = sqrt(2m+3) mu P_mm,
    P_nm = a_nm (mu P_{n-1,m} - b_nm P_{n-2,m}).
    """
    mu = np.asarray(mu, dtype=float)
    t = trunc
    s = np.sqrt((1.0 - mu) * (1.0 + mu))
    m = np.arange(t + 1, dtype=float)
    # log |P_mm| to avoid overflow/underflow in the product before the sin^m factor
    lfac = np.concatenate([[0.0], np.cumsum(np.log((2 * m[1:] - 1) / (2 * m[1:])))])
    logpmm = 0.5 * (np.log((2 * m + 1) / (4 * np.pi)) + lfac)[:, None] + m[:, None] * np.log(
        np.where(s > 0, s, 1e-300)
    )[None, :]
    sign = np.where(np.arange(t + 1) % 2 == 0, 1.0, -1.0)[:, None]
    pmm = sign * np.exp(logpmm)
    moff = m_offsets(t)
    c = moff[-1]
    ptab = np.zeros((c, mu.size))
    htab = np.zeros((c, mu.size))
    mi = np.arange(t + 1)
    prev2 = None
    prev1 = pmm
    ptab[moff[mi]] = pmm
    for l in range(1, t + 1):
        mm = mi[: t + 1 - l]
        n = mm + l
        nf = n.astype(float)
        mf = mm.astype(float)
        a = np.sqrt((4 * nf * nf - 1) / (nf * nf - mf * mf))[:, None]
        if l == 1:
            cur = a * mu[None, :] * prev1[: t + 1 - l]
        else:
            b = np.sqrt(((nf - 1) ** 2 - mf * mf) / (4 * (nf - 1) ** 2 - 1))[:, None]
            cur = a * (mu[None, :] * prev1[: t + 1 - l] - b * prev2[: t + 1 - l])
        ptab[moff[mm] + l] = cur
        prev2, prev1 = prev1, cur
    m_of, n_of = spectral_index(t)
    nf = n_of.astype(float)
    mf = m_of.astype(float)
    htab[:] = -nf[:, None] * mu[None, :] * ptab
    has_prev = n_of > m_of
    e = np.sqrt((nf * nf - mf * mf) * (2 * nf + 1) / np.maximum(2 * nf - 1, 1.0))
    idx = np.nonzero(has_prev)[0]
    htab[idx] += e[idx, None] * ptab[idx - 1]
    return ptab, htab


ROW_PAD = 8  # must equal kRowPad in csrc/internal.cuh


@dataclass(frozen=True)
class DeviceTables:
    """Legendre tables packed for the device GEMMs.

    For each m the L = T+1-m rows are parity-sorted: ``Le`` rows with n - m even
    (padded to a multiple of ``ROW_PAD`` = 8) followed by ``Lo`` rows with n - m
    odd (padded likewise), so every 8-row tile of the analysis GEMM has a single
    parity class; each row holds the ``nlat/2`` northern latitudes.  Row
    ``rowoff[m] + r`` of ``p``/``h`` is the table row, ``row_n[rowoff[m] + r]``
    its degree n (-1 for padding rows).
    """

    p: np.ndarray
    h: np.ndarray
    rowoff: np.ndarray  # int32 [T+2]
    n_even4: np.ndarray  # int32 [T+1], padded even-row count (multiple of ROW_PAD)
    row_n: np.ndarray  # int32 [rows]


def pack_device_tables(grid, ptab_north, htab_north):
    t = grid.trunc
    j = grid.nlat // 2
    moff = m_offsets(t)
    rowoff = [0]
    even4 = []
    row_n = []
    for m in range(t + 1):
        length = t + 1 - m
        le, lo = (length + 1) // 2, length // 2
        le4, lo4 = -(-le // ROW_PAD) * ROW_PAD, -(-lo // ROW_PAD) * ROW_PAD
        even4.append(le4)
        ns = [m + 2 * i for i in range(le)] + [-1] * (le4 - le)
        ns += [m + 1 + 2 * i for i in range(lo)] + [-1] * (lo4 - lo)
        row_n.extend(ns)
        rowoff.append(rowoff[-1] + le4 + lo4)
    rows = rowoff[-1]
    p = np.zeros((rows, j))
    h = np.zeros((rows, j))
    row_n = np.array(row_n, dtype=np.int32)
    valid = row_n >= 0
    m_of_row = np.repeat(np.arange(t + 1), np.diff(rowoff))
    src = moff[m_of_row[valid]] + (row_n[valid] - m_of_row[valid])
    p[valid] = ptab_north[src]
    h[valid] = htab_north[src]
    return DeviceTables(
        p=np.ascontiguousarray(p),
        h=np.ascontiguousarray(h),
        rowoff=np.array(rowoff, dtype=np.int32),
        n_even4=np.array(even4, dtype=np.int32),
        row_n=row_n,
    )


class HostTransforms:
    """Plain numpy synthesis used only for workload setup (initial-condition scaling)."""

    def __init__(self, grid):
        self.grid = grid
        self.mu, self.w = gaussian_latitudes(grid.nlat)
        self.ptab, self.htab = legendre_tables(grid.trunc, self.mu)
        self.m_of, self.n_of = spectral_index(grid.trunc)

    def _fourier(self, coef, tab):
        t = self.grid.trunc
        out = np.zeros((self.grid.nlat, self.grid.nlon // 2 + 1), dtype=complex)
        moff = m_offsets(t)
        for m in range(t + 1):
            sl = slice(moff[m], moff[m + 1])
            out[:, m] = coef[sl] @ tab[sl]
        return out

    def to_grid(self, fourier):
        return np.fft.irfft(fourier * self.grid.nlon, n=self.grid.nlon, axis=1)

    def wind(self, zeta, delta):
        """Physical (u, v) on the grid from vorticity/divergence coefficients."""
        a = self.grid.radius
        lam = self.n_of * (self.n_of + 1.0)
        inv = np.zeros_like(lam)
        inv[lam > 0] = -(a * a) / lam[lam > 0]
        psi, chi = zeta * inv, delta * inv
        im = 1j * self.m_of
        uf = (self._fourier(im * chi, self.ptab) - self._fourier(psi, self.htab)) / a
        vf = (self._fourier(im * psi, self.ptab) + self._fourier(chi, self.htab)) / a
        cosphi = np.sqrt(1.0 - self.mu**2)[:, None]
        return self.to_grid(uf) / cosphi, self.to_grid(vf) / cosphi


def random_initial_state(grid, seed, max_wind=20.0, div_ratio=0.1, slope=-1.5, transforms=None):
    """Seeded BASELINE initial state.

    Draw order with ``numpy.random.default_rng(seed)``: real parts of zeta (C),
    imaginary parts of zeta (C), real parts of delta (C), imaginary parts of
    delta (C), all standard normal.  Coefficients are multiplied by n^slope
    (amplitude ~ n^-1.5, energy ~ n^-3), n = 0 is zeroed, imag(m = 0) is
    zeroed, delta is scaled by ``div_ratio``; finally zeta and delta are scaled
    together so that max |V| over the Gaussian grid is ``max_wind``.
    Phi' starts at zero.
    """
    c = grid.n_coef
    rng = np.random.default_rng(seed)
    zr, zi, dr, di = (rng.standard_normal(c) for _ in range(4))
    m_of, n_of = spectral_index(grid.trunc)
    amp = np.zeros(c)
    amp[n_of > 0] = n_of[n_of > 0].astype(float) ** slope
    zeta = (zr + 1j * zi) * amp
    delta = div_ratio * (dr + 1j * di) * amp
    zeta[m_of == 0] = zeta[m_of == 0].real
    delta[m_of == 0] = delta[m_of == 0].real
    tr = transforms if transforms is not None else HostTransforms(grid)
    u, v = tr.wind(zeta, delta)
    scale = max_wind / np.sqrt(u * u + v * v).max()
    state = np.zeros(3 * c, dtype=complex)
    state[c : 2 * c] = zeta * scale
    state[2 * c :] = delta * scale
    return state
