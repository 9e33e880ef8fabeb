r"""CPU restatement of the reference's planar shallow-water problem.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Pinned against the
reference itself: ``tests/golden/planar.npz`` holds f_E / f_I / solve outputs
and dsdc / serial-SDC trajectories computed by ``parsdc.problems.PlanarShallowWater``
(``tests/golden/make_golden_planar.py``); ``tests/test_oracle_planar.py``
checks this module against them (f_I and the solve bitwise, f_E to FFT
rounding).

Restated, per ``pkg/src/parsdc/problems/swe.py``:

* wavenumbers, Laplacian symbol and the strict 2/3 mask  <- ``swe.py:100-125``
* ``f_impl``          <- ``swe.py:157-163``  (-Phibar delta, 0, k^2 Phi')
* ``implicit_solve``  <- ``swe.py:165-172``  per-mode 2x2 Helmholtz solve
* ``f_expl``          <- ``swe.py:174-196``  flux form with the kinetic-energy term
* velocity            <- ``swe.py:200-205``  psi = -zeta/k^2, chi = -delta/k^2

numpy.fft (pocketfft) stands in for scipy.fft; both are unnormalised forward /
1/N^2 inverse, so f_E agrees with the reference to FFT rounding.
"""

import numpy as np

from paper_2403_20135_b200.core import SplitProblem


class PlanarShallowWaterOracle(SplitProblem):
    def __init__(self, n_grid, domain_length, mean_geopotential, coriolis, hyperviscosity=0.0):
        super().__init__()
        n = int(n_grid)
        self.n_grid = n
        self.domain_length = float(domain_length)
        self.phibar = self.mean_geopotential = float(mean_geopotential)
        self.coriolis = float(coriolis)
        self.nu = float(hyperviscosity)
        d = self.domain_length / n
        kx = (2.0 * np.pi * np.fft.fftfreq(n, d=d))[:, None]
        ky = (2.0 * np.pi * np.fft.rfftfreq(n, d=d))[None, :]
        self.ikx, self.iky = 1j * kx, 1j * ky
        self.k2 = kx**2 + ky**2
        self.inv_k2 = np.zeros_like(self.k2)
        self.inv_k2[self.k2 > 0.0] = 1.0 / self.k2[self.k2 > 0.0]
        keep = (n - 1) // 3
        ix = np.rint(kx[:, 0] / (2.0 * np.pi / self.domain_length))
        iy = np.rint(ky[0, :] / (2.0 * np.pi / self.domain_length))
        self.mask = (np.abs(ix)[:, None] <= keep) & (np.abs(iy)[None, :] <= keep)
        self.shape = (n, n // 2 + 1)
        self.state_size = 3 * n * (n // 2 + 1)

    def views(self, state):
        s = state.reshape((3,) + self.shape)
        return s[0], s[1], s[2]

    def _phys(self, spec):
        return np.fft.irfft2(spec, s=(self.n_grid, self.n_grid))

    def _f_impl(self, state):
        phi, _, delta = self.views(state)
        out = np.empty((3,) + self.shape, dtype=complex)
        out[0] = -self.phibar * delta
        out[1] = 0.0
        out[2] = self.k2 * phi
        return out.reshape(-1)

    def _implicit_solve(self, alpha, beta, guess):
        bp, bz, bd = self.views(beta)
        out = np.empty((3,) + self.shape, dtype=complex)
        den = 1.0 + alpha**2 * self.phibar * self.k2
        out[0] = (bp - alpha * self.phibar * bd) / den
        out[1] = bz
        out[2] = bd + alpha * self.k2 * out[0]
        return out.reshape(-1)

    def _f_expl(self, state):
        phi, zeta, delta = self.views(state)
        psi, chi = -zeta * self.inv_k2, -delta * self.inv_k2
        u = self._phys(-self.iky * psi + self.ikx * chi)
        v = self._phys(self.ikx * psi + self.iky * chi)
        q = self.coriolis + self._phys(zeta)
        ph = self._phys(phi)
        fx, fy = np.fft.rfft2(q * u), np.fft.rfft2(q * v)
        ke = np.fft.rfft2(0.5 * (u * u + v * v))
        mx, my = np.fft.rfft2(ph * u), np.fft.rfft2(ph * v)
        out = np.empty((3,) + self.shape, dtype=complex)
        out[0] = -(self.ikx * mx + self.iky * my)
        out[1] = -(self.ikx * fx + self.iky * fy)
        out[2] = (self.ikx * fy - self.iky * fx) + self.k2 * ke
        if self.nu > 0.0:
            damp = self.nu * self.k2**2
            out[0] -= damp * phi
            out[1] -= damp * zeta
            out[2] -= damp * delta
        out *= self.mask
        return out.reshape(-1)


def relative_l2_fields(a, b):
    """Per-field relative L2 difference of two planar states (3 fields)."""
    a3, b3 = a.reshape(3, -1), b.reshape(3, -1)
    return [float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)) for x, y in zip(a3, b3)]
