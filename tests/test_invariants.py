"""Conservation of mass, energy, angular momentum and potential enstrophy by the
spherical operator under the reference's dSDC integrator (tests/sphere_invariants.py):
the CPU oracle here; the GPU path over full BASELINE runs in test_gpu_invariants.py.
The mutation cases show that the bounds would catch a wrong sign in any term of the
wind synthesis or of the divergence / curl analysis (m > 0 terms included)."""

import numpy as np
import pytest

from oracle import sdc as osdc
from oracle.sphere_swe import SphericalShallowWaterFast, SphericalShallowWaterOracle
from paper_2403_20135_b200 import CollocationTable, random_initial_state
from paper_2403_20135_b200.sphere import SphereGrid, grid_for
from sphere_invariants import BOUNDS, drifts

_TERMS = ("U_chi_P", "U_psi_H", "V_psi_P", "V_chi_H", "div_X_P", "div_Y_H", "curl_Y_P", "curl_X_H")


def _mutant(flip):
    sign = {k: (-1.0 if k == flip else 1.0) for k in _TERMS}

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

        def div_curl(self, xf, yf, weight):
            im = 1j * self.m_of
            a = self.radius
            wt = weight / self.coslat2
            div = (sign["div_X_P"] * im * self.legendre_analysis(xf, self.p, wt)
                   - sign["div_Y_H"] * self.legendre_analysis(yf, self.h, wt)) / a
            curl = (sign["curl_Y_P"] * im * self.legendre_analysis(yf, self.p, wt)
                    + sign["curl_X_H"] * self.legendre_analysis(xf, self.h, wt)) / a
            return div, curl

    return Mutant


def test_oracle_conserves_the_invariants_over_a_run():
    g = grid_for(63)
    p = SphericalShallowWaterFast(g.trunc, g.nlat, g.nlon)
    table = CollocationTable.radau_right(3)
    u0 = random_initial_state(g, seed=1)
    u = u0
    for _ in range(50):
        u = osdc.dsdc(p, u, 120.0, table, 3)
    d = drifts(p, u0, u)
    print(d)
    for k, bound in BOUNDS.items():
        assert d[k] <= bound, (k, d)


@pytest.mark.parametrize("flip", _TERMS)
def test_a_wrong_sign_breaks_energy_conservation(flip):
    g = SphereGrid(trunc=42, nlat=64, nlon=128)
    good = SphericalShallowWaterOracle(g.trunc, g.nlat, g.nlon)
    bad = _mutant(flip)(g.trunc, g.nlat, g.nlon, tables=(good.mu, good.w, good.p, good.h, good.m_of, good.n_of))
    table = CollocationTable.radau_right(3)
    u0 = random_initial_state(g, seed=1)
    u = u0
    for _ in range(6):
        u = osdc.dsdc(bad, u, 120.0, table, 3)
    d = drifts(good, u0, u)
    assert np.isfinite(list(d.values())).all()
    assert max(d["energy"] / BOUNDS["energy"], d["angular_momentum"] / BOUNDS["angular_momentum"],
               d["potential_enstrophy"] / BOUNDS["potential_enstrophy"]) > 1e2, d
    print(flip, d)
