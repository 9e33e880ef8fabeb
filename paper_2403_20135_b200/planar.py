"""CUDA-backed planar shallow water: the reference's own problem on the GPU.

``PlanarShallowWater`` restates ``parsdc.problems.PlanarShallowWater``
(``pkg/src/parsdc/problems/swe.py:57-205``): doubly periodic f-plane shallow
water in vorticity-divergence form, state = three rfft2 spectra
``(Phi', zeta, delta)`` of shape ``[N][N/2 + 1]``, implicit gravity-wave part
``L_g = (-Phibar delta, 0, k^2 Phi')`` and the flux-form explicit tendency with
2/3 dealiasing.  f_E runs as three CUDA kernels (``csrc/planar.cu``); f_I, the
implicit solve and the sweep kernels are the same bit-exact node kernels the
spherical problem uses, with ``lam = k^2``.  Because this problem exists in
the reference, the GPU path is pinned end to end against vectors produced by
the reference itself (``tests/golden/make_golden_planar.py``).

Host-side helpers (wavenumbers, mask, views, diagnostics, the balanced-jet
initial condition) restate the reference's construction with numpy; they are
not on the hot path.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ParameterError, ValidationError
from .problem import DeviceProblem


class PlanarShallowWater(DeviceProblem):
    """Pseudo-spectral planar shallow water on one B200 (reference constructor signature).

    ``space_threads`` is accepted for drop-in compatibility and ignored (the
    device decides its own parallelism); ``device`` and ``max_batch`` are the
    GPU extras."""

    def __init__(self, n_grid, domain_length, mean_geopotential, coriolis, hyperviscosity=0.0,
                 space_threads=1, device=0, max_batch=8):
        super().__init__()
        import torch

        # validation as problems/swe.py:87-98
        if not isinstance(n_grid, (int, np.integer)) or n_grid < 8 or n_grid % 2:
            raise ParameterError(f"n_grid must be an even integer >= 8, got {n_grid!r}")
        if domain_length <= 0.0:
            raise ParameterError("domain_length must be positive")
        if mean_geopotential <= 0.0:
            raise ParameterError("mean_geopotential must be positive")
        if hyperviscosity < 0.0:
            raise ParameterError("hyperviscosity must be non-negative")
        if not isinstance(space_threads, (int, np.integer)) or space_threads < 1:
            raise ParameterError("space_threads must be a positive integer")
        if max_batch < 1:
            raise ParameterError("max_batch must be positive")
        self.n_grid = int(n_grid)
        self.domain_length = float(domain_length)
        self.mean_geopotential = float(mean_geopotential)
        self.phibar = self.mean_geopotential
        self.coriolis = float(coriolis)
        self.hyperviscosity = float(hyperviscosity)
        self.space_threads = int(space_threads)
        self.max_batch = int(max_batch)

        n = self.n_grid
        spacing = self.domain_length / n
        self.wavenumbers_x = 2.0 * np.pi * np.fft.fftfreq(n, d=spacing)
        self.wavenumbers_y = 2.0 * np.pi * np.fft.rfftfreq(n, d=spacing)
        kx = self.wavenumbers_x[:, None]
        ky = self.wavenumbers_y[None, :]
        self._ikx = 1j * kx
        self._iky = 1j * ky
        self.laplacian_symbol = kx**2 + ky**2
        # strict 2/3 rule (keep < N/3)
        keep = (n - 1) // 3
        index_x = np.rint(self.wavenumbers_x / (2.0 * np.pi / self.domain_length))
        index_y = np.rint(self.wavenumbers_y / (2.0 * np.pi / self.domain_length))
        self.dealias_mask = (np.abs(index_x)[:, None] <= keep) & (np.abs(index_y)[None, :] <= keep)
        self._spectral_shape = (n, n // 2 + 1)
        self.n_coef = n * (n // 2 + 1)
        self.state_size = 3 * self.n_coef
        self.lam = np.ascontiguousarray(self.laplacian_symbol.reshape(-1))

        self._lib = _native.lib()
        self.device = torch.device("cuda", device)
        cfg = _native.PlanarConfig(n_grid=n, max_batch=self.max_batch,
                                   domain_length=self.domain_length,
                                   mean_geopotential=self.mean_geopotential,
                                   coriolis=self.coriolis, hyperviscosity=self.hyperviscosity)
        kxa = np.ascontiguousarray(self.wavenumbers_x)
        kya = np.ascontiguousarray(self.wavenumbers_y)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(
                self._lib.sdcsw_plan_create_planar(device, ctypes.byref(cfg), _native.dptr(kxa),
                                                   _native.dptr(kya), _native.dptr(self.lam),
                                                   ctypes.byref(handle)),
                "sdcsw_plan_create_planar",
            )
        self._plan = handle

    def solve_coefficients(self, alpha):
        """(alpha Phibar, alpha**2 Phibar): the reference's own expressions
        (problems/swe.py:168-170; Python's ``alpha**2`` is not always ``alpha*alpha``)."""
        return alpha * self.mean_geopotential, alpha**2 * self.mean_geopotential

    @property
    def n_dof(self):
        return self.n_grid**2

    # -- state layout (problems/swe.py:135-147) ---------------------------------

    def spectral_views(self, state):
        n, nh = self._spectral_shape
        stacked = state.reshape(3, n, nh)
        return stacked[0], stacked[1], stacked[2]

    def pack(self, phi, zeta, delta):
        out = np.empty((3,) + self._spectral_shape, dtype=complex)
        out[0], out[1], out[2] = phi, zeta, delta
        return out.reshape(self.state_size)

    # -- host diagnostics (problems/swe.py:207-250) -----------------------------

    def _to_physical(self, spec):
        n = self.n_grid
        return np.fft.irfft2(spec, s=(n, n))

    def _velocity(self, zeta, delta):
        inv = np.zeros_like(self.laplacian_symbol)
        nz = self.laplacian_symbol > 0.0
        inv[nz] = 1.0 / self.laplacian_symbol[nz]
        psi = -zeta * inv
        chi = -delta * inv
        u = self._to_physical(-self._iky * psi + self._ikx * chi)
        v = self._to_physical(self._ikx * psi + self._iky * chi)
        return u, v

    def velocity_from_state(self, state):
        _, zeta, delta = self.spectral_views(state)
        scale = max(np.linalg.norm(zeta), np.linalg.norm(delta), 1.0)
        for name, field in (("vorticity", zeta), ("divergence", delta)):
            if abs(field[0, 0]) > 1e-12 * scale:
                raise ValidationError(f"mean {name} mode must vanish, got {field[0, 0]!r}")
        return self._velocity(zeta, delta)

    def vorticity_physical(self, state):
        _, zeta, _ = self.spectral_views(state)
        return self._to_physical(zeta)

    def error_field(self, state):
        return self.vorticity_physical(state)

    def mean_geopotential_anomaly(self, state):
        phi, _, _ = self.spectral_views(state)
        return phi[0, 0].real / self.n_grid**2

    def total_energy(self, state):
        phi, zeta, delta = self.spectral_views(state)
        u, v = self._velocity(zeta, delta)
        phi_phys = self._to_physical(phi)
        kinetic = 0.5 * (self.mean_geopotential + phi_phys) * (u * u + v * v)
        return float(np.mean(kinetic + 0.5 * phi_phys**2))


@dataclass(frozen=True)
class JetConfig:
    """Balanced zonal jet parameters (as the reference's ``JetConfig``)."""

    u_max: float = 80.0
    y_center: float = None
    width: float = None
    perturbation_amplitude: float = 1e-4
    perturbation_wavenumber: int = 3


def jet_initial_condition(problem, config=None):
    """Geostrophically balanced zonal jet u(y) = u_max sech^2((y - y0)/w) with an
    optional meridional-velocity perturbation; Phi' solves dPhi'/dy = -f0 u
    spectrally with zero mean (the construction of problems/swe.py:346-400)."""
    config = JetConfig() if config is None else config
    length = problem.domain_length
    y0 = length / 2.0 if config.y_center is None else config.y_center
    width = length / 15.0 if config.width is None else config.width
    if width <= 0.0 or config.u_max <= 0.0:
        raise ParameterError("jet width and peak velocity must be positive")
    n = problem.n_grid
    coords = np.arange(n) * length / n
    x, y = coords[:, None], coords[None, :]
    u_phys = np.broadcast_to(config.u_max / np.cosh((y - y0) / width) ** 2, (n, n))
    v_phys = (config.perturbation_amplitude * config.u_max
              * np.cos(2.0 * np.pi * config.perturbation_wavenumber * x / length)
              * np.exp(-(((y - y0) / width) ** 2)))
    u_hat = np.fft.rfft2(np.ascontiguousarray(u_phys)) * problem.dealias_mask
    v_hat = np.fft.rfft2(v_phys) * problem.dealias_mask
    zeta = problem._ikx * v_hat - problem._iky * u_hat
    delta = problem._ikx * u_hat + problem._iky * v_hat
    zeta[0, 0] = 0.0
    delta[0, 0] = 0.0
    ky = np.broadcast_to(problem.wavenumbers_y[None, :], u_hat.shape)
    phi = np.zeros_like(u_hat)
    nz = ky != 0.0
    phi[nz] = -problem.coriolis * u_hat[nz] / (1j * ky[nz])
    return problem.pack(phi, zeta, delta)
