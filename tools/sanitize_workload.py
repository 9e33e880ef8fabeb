"""Workload for compute-sanitizer (memcheck / synccheck / racecheck / initcheck): every
stage-kernel family of the path at small sizes, a few steps each, eager launches and one
graph replay.  Run on the GPU box as

    compute-sanitizer --tool memcheck python tools/sanitize_workload.py [part ...]

Parts: latency (T63/T127 fused, unfused, chained, sequential, serial, hooked, residual),
hfree (T127 ensemble plans and T255: the table-streaming H-free transforms, batch tails the
round-1 advisor asked for), planar.  Default: all.

compute-sanitizer is closed on this round's GPU pool (every tool exits at once with "closed on
this pool"; gpurun of 2026-10-21), so this script has only run plain there (all parts finite);
its stand-in is the library's own canary check: SDCSW_GUARD=1 python tools/sanitize_workload.py
prints the canary bytes overwritten after every part (tests/test_gpu_guard.py asserts 0)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_20135_b200 import (  # noqa: E402
    CollocationTable, SdcConfig, SweepMode, random_initial_state,
)
from paper_2403_20135_b200.integrators import DeviceStepper  # noqa: E402
from paper_2403_20135_b200.planar import PlanarShallowWater, jet_initial_condition  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402


def cfg_for(m, mode=SweepMode.DIAGONAL_PARALLEL):
    return SdcConfig(table=CollocationTable.radau_right(m), n_sweeps=m, mode=mode)


def dev_state(p, u0):
    return p._to_device(u0).reshape(-1).contiguous()


def finite(t):
    return bool(torch.isfinite(torch.view_as_real(t) if t.is_complex() else t).all())


def latency():
    for trunc, m, dt in ((63, 3, 120.0), (127, 4, 90.0)):
        p = SphericalShallowWater(trunc, max_batch=8)
        u0 = random_initial_state(p.grid, 1)
        for serial in (False, True):
            mode = SweepMode.SERIAL if serial else SweepMode.DIAGONAL_PARALLEL
            st = DeviceStepper(p, cfg_for(m, mode), dt, serial=serial)
            u = dev_state(p, u0)
            st.run(u, 2, use_graph=False)
            st.run(u, 8, use_graph=True)
            seen = []
            st.step_hooked(u, lambda k, s: seen.append(k))
            st.profile_step(u)
            if not serial:
                st.set_fused(False)
                st.set_chains(2)
                st.run(u, 1, use_graph=False)
                st.set_chains(1)
                st.set_sequential(True)
                st.run(u, 1, use_graph=False)
            torch.cuda.synchronize()
            print(f"T{trunc} serial={serial} finite={finite(u)} hooks={len(seen)}", flush=True)
            st.close()
        big = p.empty_states(8)
        src = torch.from_numpy(np.stack([u0] * 8)).to(p.device).contiguous()
        p.f_expl_device(src, big, 8)
        p.f_expl_device(src, big, 5)
        torch.cuda.synchronize()
        p.close()


def hfree():
    # ensemble-sized T127 plans: bulk synthesis in batch blocks with partial tails
    base = None
    for nb in (16, 25, 256):  # 256 = the c4 batch (64 members x 4 nodes), 256 % 6 = 4
        p = SphericalShallowWater(127, max_batch=nb)
        assert p.uses_ponly
        if base is None:
            base = [random_initial_state(p.grid, b) for b in range(25)]
        st = np.stack([base[b % 25] for b in range(nb)])
        u = torch.from_numpy(st).to(p.device)
        o = p.empty_states(nb)
        for n in (nb, nb - 3, 1):
            p.f_expl_device(u, o, n)
        torch.cuda.synchronize()
        print(f"T127 H-free f_E max_batch={nb} finite={finite(o)}", flush=True)
        if nb == 16:
            ens = torch.from_numpy(st[:4]).to(p.device).contiguous()
            s = DeviceStepper(p, cfg_for(4), 90.0, serial=False, members=4)
            s.run(ens, 1, use_graph=False)
            s.run(ens, 2, use_graph=True)
            torch.cuda.synchronize()
            print(f"T127 4-member ensemble dSDC finite={finite(ens)}", flush=True)
            s.close()
        p.close()
    # T255: table-streaming single-member dSDC (H-free node kernel) and serial SDC
    p = SphericalShallowWater(255, max_batch=8)
    assert p.uses_ponly
    u0 = random_initial_state(p.grid, 2)
    for serial in (False, True):
        mode = SweepMode.SERIAL if serial else SweepMode.DIAGONAL_PARALLEL
        s = DeviceStepper(p, cfg_for(4, mode), 60.0, serial=serial)
        u = dev_state(p, u0)
        s.run(u, 1, use_graph=False)
        s.run(u, 2, use_graph=True)
        if not serial:
            s.set_chains(2)
            s.run(u, 1, use_graph=False)
            s.set_chains(1)
            s.set_sequential(True)
            s.run(u, 1, use_graph=False)
        torch.cuda.synchronize()
        print(f"T255 serial={serial} finite={finite(u)}", flush=True)
        s.close()
    p.close()


def planar():
    pl = PlanarShallowWater(64, 4.0e6, 1.0e5, 1.0e-4, max_batch=4)
    x = jet_initial_condition(pl)
    st = DeviceStepper(pl, cfg_for(3), 60.0, serial=False)
    u = dev_state(pl, x)
    st.run(u, 2, use_graph=False)
    torch.cuda.synchronize()
    print(f"planar finite={finite(u)}", flush=True)
    st.close()


def guard_report():
    """Canary bytes overwritten so far (SDCSW_GUARD=1; include/sdcsw.h sdcsw_guard_check)."""
    import ctypes

    from paper_2403_20135_b200 import _native

    bad, live = ctypes.c_longlong(), ctypes.c_int()
    _native.check(_native.lib().sdcsw_guard_check(ctypes.byref(bad), ctypes.byref(live)), "guard")
    return bad.value, live.value


if __name__ == "__main__":
    parts = sys.argv[1:] or ["latency", "hfree", "planar"]
    for name in parts:
        {"latency": latency, "hfree": hfree, "planar": planar}[name]()
        print(f"guard after {name}: corrupted_bytes={guard_report()[0]}", flush=True)
    if os.environ.get("SDCSW_GUARD") == "1":
        from paper_2403_20135_b200 import _native

        before = guard_report()[0]
        _native.check(_native.lib().sdcsw_guard_selftest(), "selftest")
        print(f"guard selftest: +{guard_report()[0] - before} corrupted byte(s)", flush=True)
    print("sanitize workload done", flush=True)
