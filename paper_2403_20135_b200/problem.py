"""CUDA-backed spherical shallow-water ``SplitProblem`` (the drop-in problem).

``SphericalShallowWater`` implements the reference contract
(``pkg/src/parsdc/core.py:85-126``) with numpy in/out, so it runs unmodified
under the reference's own ``dsdc_step`` / ``integrate``; every evaluation is
one call into ``libsdcsw.so`` (no CPU fallback).  The device-resident methods
(``*_device``) take and return torch CUDA tensors and are what the fused
steppers in :mod:`.integrators` use.

The spherical formulation restates the planar template
(``pkg/src/parsdc/problems/swe.py:157-205``) as documented in DESIGN.md and
SURVEY.md Appendix A: state ``(Phi', zeta, delta)`` spectral coefficients,
implicit part ``L_g = (-Phibar delta, 0, n(n+1)/a^2 Phi')``, explicit part the
flux-form advection, Coriolis and kinetic-energy terms.
"""

import ctypes

import numpy as np

from . import _native
from .core import SplitProblem
from .errors import ParameterError
from .sphere import (
    EARTH_RADIUS,
    GRAVITY,
    MEAN_DEPTH,
    OMEGA,
    SphereGrid,
    gaussian_latitudes,
    grid_for,
    laplacian_eigenvalues,
    legendre_tables,
    pack_device_tables,
    spectral_index,
)


class DeviceProblem(SplitProblem):
    """Plumbing shared by the CUDA problems: the plan handle, device-resident
    operations on torch complex128 tensors, and the numpy ``SplitProblem``
    contract on top of them (one C-ABI call per evaluation, no CPU fallback).

    Subclasses set ``_lib``, ``_plan``, ``device``, ``state_size``,
    ``max_batch`` and ``mean_geopotential``."""

    # -- lifecycle ------------------------------------------------------------

    def close(self):
        if getattr(self, "_plan", None):
            self._lib.sdcsw_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def uses_ponly(self):
        """True when f_E runs the H-free transforms (``sdcsw_plan_transform_kind``)."""
        kind, rows = ctypes.c_int(), ctypes.c_int()
        _native.check(self._lib.sdcsw_plan_transform_kind(self._plan, ctypes.byref(kind), ctypes.byref(rows)),
                      "sdcsw_plan_transform_kind")
        return kind.value == 1

    @property
    def handle(self):
        return self._plan

    def stream(self):
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    # -- device-resident operations (torch complex128 tensors) ----------------

    def empty_states(self, nb):
        import torch

        return torch.empty((nb, self.state_size), dtype=torch.complex128, device=self.device)

    def _check_batch(self, t, nb):
        if t.dtype.__str__() != "torch.complex128" or not t.is_contiguous() or t.device != self.device:
            raise ParameterError("device states must be contiguous complex128 tensors on the plan's device")
        if t.numel() < nb * self.state_size:
            raise ParameterError("tensor too small for the requested batch")

    def f_expl_device(self, u, out, nb=None):
        nb = u.shape[0] if nb is None else nb
        if nb > self.max_batch:
            raise ParameterError(f"batch {nb} exceeds max_batch {self.max_batch}")
        self._check_batch(u, nb)
        self._check_batch(out, nb)
        _native.check(
            self._lib.sdcsw_f_expl(self._plan, u.data_ptr(), out.data_ptr(), nb, self.stream()),
            "sdcsw_f_expl",
        )
        return out

    def workspace(self, which):
        """A float64 torch view (no copy) of internal workspace ``which``
        (``sdcsw_workspace``: 0 = Fourier coefficients, 1 = analysis data);
        for tests and diagnostics."""
        import torch

        ptr, nbytes = ctypes.c_void_p(), ctypes.c_longlong()
        _native.check(self._lib.sdcsw_workspace(self._plan, which, ctypes.byref(ptr), ctypes.byref(nbytes)),
                      "sdcsw_workspace")

        class _View:
            __cuda_array_interface__ = {"shape": (nbytes.value // 8,), "typestr": "<f8",
                                        "data": (ptr.value, False), "version": 3, "strides": None}

        return torch.as_tensor(_View(), device=self.device)

    def f_impl_device(self, u, out, nb=None):
        nb = u.shape[0] if nb is None else nb
        self._check_batch(u, nb)
        self._check_batch(out, nb)
        _native.check(
            self._lib.sdcsw_f_impl(self._plan, u.data_ptr(), out.data_ptr(), nb, self.stream()),
            "sdcsw_f_impl",
        )
        return out

    def solve_coefficients(self, alpha):
        """(alpha*Phibar, alpha*alpha*Phibar): same Python expressions as the oracle."""
        return alpha * self.mean_geopotential, alpha * alpha * self.mean_geopotential

    def implicit_solve_device(self, alphas, beta, out):
        nb = len(alphas)
        self._check_batch(beta, nb)
        self._check_batch(out, nb)
        coef = np.empty((nb, 3))
        for b, a in enumerate(alphas):
            a = float(a)
            coef[b] = (a,) + self.solve_coefficients(a)
        _native.check(
            self._lib.sdcsw_implicit_solve(self._plan, _native.dptr(coef), beta.data_ptr(),
                                           out.data_ptr(), nb, self.stream()),
            "sdcsw_implicit_solve",
        )
        return out

    # -- SplitProblem contract (numpy in / out) --------------------------------

    def _to_device(self, state):
        import torch

        arr = np.ascontiguousarray(state, dtype=np.complex128).reshape(-1)
        if arr.size != self.state_size:
            raise ParameterError(f"state has {arr.size} entries, expected {self.state_size}")
        return torch.from_numpy(arr).to(self.device).reshape(1, -1)

    def _to_host(self, t):
        return t.reshape(-1).cpu().numpy().copy()

    def _f_expl(self, state):
        u = self._to_device(state)
        out = self.empty_states(1)
        return self._to_host(self.f_expl_device(u, out, 1))

    def _f_impl(self, state):
        u = self._to_device(state)
        out = self.empty_states(1)
        return self._to_host(self.f_impl_device(u, out, 1))

    def _implicit_solve(self, alpha, beta, guess):
        b = self._to_device(beta)
        out = self.empty_states(1)
        return self._to_host(self.implicit_solve_device([alpha], b, out))



class SphericalShallowWater(DeviceProblem):
    """Rotating shallow water on the sphere, T-truncated spherical harmonics, on one B200.

    Parameters
    ----------
    trunc : int
        Triangular truncation T.
    nlat, nlon : int, optional
        Gaussian grid; defaults to the BASELINE grids (T63 192x96 ... T511 1536x768).
    device : int
        CUDA device ordinal.
    max_batch : int
        Largest number of states one batched call may carry (nodes x members).
    """

    def __init__(self, trunc, nlat=None, nlon=None, radius=EARTH_RADIUS, gravity=GRAVITY,
                 omega=OMEGA, mean_depth=MEAN_DEPTH, device=0, max_batch=8):
        super().__init__()
        import torch

        base = grid_for(trunc) if not (nlat and nlon) else None
        self.grid = SphereGrid(
            trunc=trunc,
            nlat=nlat or base.nlat,
            nlon=nlon or base.nlon,
            radius=float(radius),
            gravity=float(gravity),
            omega=float(omega),
            mean_depth=float(mean_depth),
        )
        if max_batch < 1:
            raise ParameterError("max_batch must be positive")
        self._lib = _native.lib()
        self.device = torch.device("cuda", device)
        self.trunc = trunc
        self.n_coef = self.grid.n_coef
        self.state_size = self.grid.state_size
        self.mean_geopotential = self.grid.mean_geopotential
        self.phibar = self.mean_geopotential
        self.max_batch = int(max_batch)
        self.m_of, self.n_of = spectral_index(trunc)
        self.lam = laplacian_eigenvalues(self.grid)

        mu, w = gaussian_latitudes(self.grid.nlat)
        half = self.grid.nlat // 2
        self.mu, self.weights = mu, w
        ptab, htab = legendre_tables(trunc, mu[:half])
        tabs = pack_device_tables(self.grid, ptab, htab)
        cfg = _native.Config(
            trunc=trunc,
            nlat=self.grid.nlat,
            nlon=self.grid.nlon,
            max_batch=self.max_batch,
            radius=self.grid.radius,
            omega=self.grid.omega,
            phibar=self.mean_geopotential,
        )
        arrays = dict(
            mu=np.ascontiguousarray(mu[:half]),
            w=np.ascontiguousarray(w[:half]),
            lam=np.ascontiguousarray(self.lam),
            p=tabs.p, h=tabs.h, rowoff=tabs.rowoff, n_even=tabs.n_even4, row_n=tabs.row_n,
        )
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _native.check(
                self._lib.sdcsw_plan_create(
                    device, ctypes.byref(cfg), _native.dptr(arrays["mu"]), _native.dptr(arrays["w"]),
                    _native.dptr(arrays["p"]), _native.dptr(arrays["h"]),
                    _native.iptr(arrays["rowoff"]), _native.iptr(arrays["n_even"]),
                    _native.iptr(arrays["row_n"]), _native.dptr(arrays["lam"]), ctypes.byref(handle),
                ),
                "sdcsw_plan_create",
            )
        self._plan = handle
        self.table_bytes = 2 * tabs.p.nbytes

    # -- layout helpers ----------------------------------------------------------

    @property
    def n_dof(self):
        return self.grid.n_dof

    def vorticity_physical(self, state):
        """Vorticity on the Gaussian grid (host synthesis; diagnostics, not the hot path)."""
        from .sphere import HostTransforms

        if getattr(self, "_host", None) is None:
            self._host = HostTransforms(self.grid)
        h = self._host
        c = self.n_coef
        zeta = np.asarray(state)[c : 2 * c]
        return h.to_grid(h._fourier(zeta, h.ptab))

    def error_field(self, state):
        """Field entering the work-precision error norm (as the planar problem's)."""
        return self.vorticity_physical(state)

    def spectral_views(self, state):
        c = self.n_coef
        return state[:c], state[c : 2 * c], state[2 * c :]
