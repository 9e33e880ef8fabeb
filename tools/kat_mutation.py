"""GPU mutation check for the m > 0 known-answer flows.

Builds libsdcsw.so with -DSDCSW_MUTATE_UCHI=1 (the i m chi term of U gets the
wrong sign in every synthesis-operand writer) into a scratch directory and
prints, as one JSON line, the worst known-answer-flow error of that library
and of the default one, plus each library's energy / potential-enstrophy drift
over 6 dSDC steps at T63 (tests/sphere_invariants.py).  ``python tools/kat_mutation.py [--eval LIB]``
(GPU; --eval is the per-library child process)."""

import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def evaluate():
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    import numpy as np

    from oracle.sphere_swe import SphericalShallowWaterOracle
    from paper_2403_20135_b200.problem import SphericalShallowWater
    from sphere_kats import field_errors, rossby_haurwitz, tilted_potential, tilted_rotation

    p = SphericalShallowWater(63, max_batch=3)
    o = SphericalShallowWaterOracle(63, p.grid.nlat, p.grid.nlon)
    out = {}
    for name, fn in (("rotation_a45", lambda o: tilted_rotation(o, np.pi / 4)),
                     ("potential_a45", lambda o: tilted_potential(o, np.pi / 4)),
                     ("potential_a90", lambda o: tilted_potential(o, np.pi / 2)),
                     ("rossby_haurwitz4", rossby_haurwitz)):
        x, want = fn(o)
        fe, fi = p.f_expl(x), p.f_impl(x)
        e = field_errors(o, fe + fi, want, [fe, fi])
        out[name] = float(max(e[:2]) if name.startswith("rossby") else max(e))
    # conservation over a short run on the device stepper (tests/sphere_invariants.py)
    import torch

    from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
    from paper_2403_20135_b200.integrators import DeviceStepper
    from sphere_invariants import drifts

    u0 = random_initial_state(p.grid, seed=1)
    cfg = SdcConfig(table=CollocationTable.radau_right(3), n_sweeps=3, mode=SweepMode.DIAGONAL_PARALLEL)
    st = DeviceStepper(p, cfg, 120.0, serial=False)
    u = torch.from_numpy(u0).to(p.device).reshape(-1).contiguous()
    st.run(u, 6, use_graph=False)
    torch.cuda.synchronize()
    d = drifts(o, u0, u.cpu().numpy())
    out["energy_drift_6_steps"] = float(d["energy"])
    out["enstrophy_drift_6_steps"] = float(d["potential_enstrophy"])
    st.close()
    p.close()
    print(json.dumps(out))


def run(lib):
    env = dict(os.environ, SDCSW_LIB_PATH=lib)
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--eval"], env=env,
                       capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    if "--eval" in sys.argv:
        return evaluate()
    tmp = tempfile.mkdtemp(prefix="sdcsw_mut_")
    try:
        csrc = os.path.join(tmp, "pkg", "csrc")
        os.makedirs(csrc)
        shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
        src = os.path.join(ROOT, "paper_2403_20135_b200", "csrc")
        for f in os.listdir(src):
            if f.endswith((".cu", ".cuh")) or f == "Makefile":
                shutil.copy(os.path.join(src, f), csrc)
        mk = os.path.join(csrc, "Makefile")
        text = open(mk).read().replace("FLAGS = ", "FLAGS = -DSDCSW_MUTATE_UCHI=1 ", 1)
        open(mk, "w").write(text)
        subprocess.run(["make", "-s", "-C", csrc, "-j8"], check=True, capture_output=True)
        mutant = run(os.path.join(tmp, "pkg", "libsdcsw.so"))
        default = run(os.path.join(ROOT, "paper_2403_20135_b200", "libsdcsw.so"))
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    print(json.dumps({"default": default, "mutant_u_chi_sign": mutant}))


if __name__ == "__main__":
    main()
