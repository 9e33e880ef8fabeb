"""Launch the stage kernels bench.py reports, on live states, inside a
cudaProfilerStart/Stop region, one labelled launch each, for
``ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum``.
Prints the labels in launch order (one per line, prefixed "LAUNCH ");
tools/traffic_to_json.py pairs them with the ncu rows and writes
profiles/ncu_traffic_r02.json.

python tools/traffic_capture.py c1 c3
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, _native, random_initial_state  # noqa: E402
from paper_2403_20135_b200.integrators import DeviceStepper, diagonal_step_coefficients  # noqa: E402
from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402


def main(names):
    jobs = []
    for name in names:
        c = bench.CONFIGS[name]
        mm, kk, me = c["nodes"], c["sweeps"], c.get("members", 1)
        # ensembles (c4): the init f_E carries the members, the sweeps nodes x members
        # states - the launches bench.py's stage roofline times
        p = SphericalShallowWater(c["trunc"], max_batch=mm * me)
        cfg = SdcConfig(table=CollocationTable.radau_right(mm), n_sweeps=kk, mode=SweepMode.DIAGONAL_PARALLEL)
        st = DeviceStepper(p, cfg, c["dt"], serial=False, members=me)
        u0 = np.stack([random_initial_state(p.grid, c["seed"] + e) for e in range(me)])
        u = torch.from_numpy(u0).to(p.device).reshape(-1).contiguous()
        st.run(u, 3)
        seq = bench.live_states(st, u, mm)
        many = torch.cat([x.reshape(me, -1) for x in seq]).contiguous()
        one = seq[0].reshape(me, -1).contiguous()
        nbm = mm * me
        fused = st.launches_per_step == 3 * kk
        out, fi = p.empty_states(nbm), p.empty_states(nbm)
        fe = p.empty_states(nbm)
        p.f_expl_device(many, fe, nbm)
        p.f_impl_device(many, fi, nbm)
        coef = diagonal_step_coefficients(cfg, c["dt"], p.mean_geopotential)
        blk = mm * (mm + 4)
        b = CudaNodeBackend(p)
        jobs.append((name, p, st, seq, many, one, me, fused, out, fi, fe, coef, blk, b, mm, kk))
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for name, p, st, seq, many, one, me, fused, out, fi, fe, coef, blk, b, mm, kk in jobs:
        lib, s = p._lib, p.stream()
        for nb, states in ((me, one), (mm * me, many)):
            def stage(k):
                dst = fi if k == 4 else out
                _native.check(lib.sdcsw_transform_stage(p.handle, k, states.data_ptr(), dst.data_ptr(), nb, s))
            # H-free plans: stage 3 = operand conversion + synthesis, stage 2 = analysis +
            # assembly (two kernels each, summed by traffic_to_json); stage 0 adds the prep
            po = p.uses_ponly
            stage(0)  # operand prep + synthesis (not labelled)
            print(f"SKIP {3 if po else 2}", flush=True)
            for k, lab in ((3, "legendre_synthesis"), (1, "ring_fft_products"), (2, "legendre_analysis")):
                stage(k)
                for _ in range(2 if po and k != 1 else 1):
                    print(f"LAUNCH {name}:{lab}:nb{nb}", flush=True)
            if fused and nb == mm * me:
                stage(4)
                print(f"LAUNCH {name}:legendre_analysis_fused:nb{nb}", flush=True)
        if me > 1:
            continue  # (the node kernels' roofline is reported for c3 only)
        uo, fo, one1 = p.empty_states(mm), p.empty_states(mm), p.empty_states(1)
        b.sweep_nodes(mm, 0, mm, np.ascontiguousarray(coef[:blk]), seq[0], fe, 1, fi, 1, False, uo, fo)
        print(f"LAUNCH {name}:sweep_nodes:nb{mm}", flush=True)
        b.final_node(mm, np.ascontiguousarray(coef[(kk - 1) * blk:]), seq[0], fe, 1, fi, 1, False, one1)
        print(f"LAUNCH {name}:final_node:nb{mm}", flush=True)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c3"])
