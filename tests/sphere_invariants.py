r"""Conserved integrals of the rotating shallow-water equations on the sphere, as an
independent check of the spherical explicit operator over its whole spectrum.

The analytic known-answer flows (tests/sphere_kats.py) are low-degree fields. These are
the conservation laws of the continuous equations (inviscid, no forcing), which hold for
any state and follow from the vector form of the equations, not from the transform
formulas of SURVEY.md Appendix A:

    mass              int Phi' dA                              (exact: Phi'_00 has no tendency)
    energy            int [ h |v|^2 / 2 + Phi'^2 / 2 ] dA      (h = Phibar + Phi'; the h-linear
                                                               part of h^2/2 is mass)
    angular momentum  int h (u cos(phi) + Omega a cos(phi)^2) a dA   (about the rotation axis)
    pot. enstrophy    int (zeta + f)^2 / (2 h) dA

A truncated spectral model conserves the last three up to truncation and time-stepping
error: measured on the CPU oracle (T63, 50 dSDC steps of 120 s, M = K = 4, n^-1.5 spectrum)
the drifts are 3e-10 / 1e-12 / 4e-9 of the scales below, while flipping the sign of any single term of
the wind synthesis or of the divergence / curl analysis moves the energy by 1e-3..1e-1 in
20 steps.  Drifts are reported relative to the kinetic energy, the relative angular
momentum int |h u cos(phi) a| dA and the relative enstrophy int zeta^2 / (2 h) dA, not to
the (much larger) planetary parts.  The diagnostics always use the unmodified oracle."""

import numpy as np


def invariants(o, state):
    """(values, scales) of the four integrals for ``state`` on the grid of oracle ``o``."""
    phi, zeta, _ = o.views(np.asarray(state))
    u, v = o.wind(state)
    pg, zg = o.synthesize(phi), o.synthesize(zeta)
    h = o.phibar + pg
    cphi = np.sqrt(o.coslat2)[:, None]
    f = (2.0 * o.omega * o.mu)[:, None]
    a = o.radius

    def integral(x):
        return a * a * (2.0 * np.pi / o.nlon) * float(np.sum(o.w[:, None] * x))

    kinetic = 0.5 * h * (u * u + v * v)
    values = {
        "mass": integral(pg),
        "energy": integral(kinetic + 0.5 * pg * pg),
        "angular_momentum": integral(h * (u * cphi + o.omega * a * cphi * cphi) * a),
        "potential_enstrophy": integral((zg + f) ** 2 / (2.0 * h)),
    }
    scales = {
        "mass": integral(h),
        "energy": integral(kinetic),
        "angular_momentum": integral(np.abs(h * u * cphi * a)),
        "potential_enstrophy": integral(zg * zg / (2.0 * h)),
    }
    return values, scales


def drifts(o, before, after):
    """Change of every integral from state ``before`` to ``after``, relative to its scale."""
    v0, s0 = invariants(o, before)
    v1, _ = invariants(o, after)
    return {k: abs(v1[k] - v0[k]) / s0[k] for k in v0}


# bounds for the BASELINE configs' runs (dSDC, M = K >= 3, omega dt <= 0.75).  The drift is
# time-stepping error: c0's third-order M = K = 3 at dt = 120 s gives 5.5e-8 / 2.9e-8 / 5.8e-7
# over 50 steps, M = K = 4 two orders less; a sign error gives 1e-3..1e-1 within 6 steps
BOUNDS = {"mass": 1e-13, "energy": 1e-6, "angular_momentum": 1e-6, "potential_enstrophy": 1e-5}
