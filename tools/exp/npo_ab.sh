#!/bin/bash
# H-free node kernel writing the operand (nodes_po) vs node states + operand kernel
cd "$(dirname "$0")/../.."
python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.problem import SphericalShallowWater
for T, M, K, E in ((255, 4, 4, 1), (127, 4, 4, 8), (511, 5, 3, 1)):
    outs = []
    for po in ("1", "0"):
        os.environ["SDCSW_NODES_PO"] = po
        p = SphericalShallowWater(T, max_batch=M * E)
        cfg = SdcConfig(table=CollocationTable.radau_right(M), n_sweeps=K, mode=SweepMode.DIAGONAL_PARALLEL)
        st = DeviceStepper(p, cfg, 60.0, serial=False, members=E)
        u0 = np.stack([random_initial_state(p.grid, 5 + e) for e in range(E)])
        u = torch.from_numpy(u0).to(0).reshape(-1).contiguous()
        st.run(u, 3)
        torch.cuda.synchronize()
        outs.append(u.cpu().numpy())
        st.close(); p.close()
    print("T", T, "E", E, "nodes_po bitwise == operand-kernel route:", np.array_equal(outs[0].view(np.uint64), outs[1].view(np.uint64)), flush=True)
PY
for r in 1 2; do
for po in 0 1; do
  SDCSW_NODES_PO=$po python tools/stage_bench.py c2 c3 2>&1 | grep "^c" | awk -v f=$po '{print "npo" f, $1, $(NF-1), $NF}'
  SDCSW_NODES_PO=$po timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-large 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('npo$po c4', round(d['value'],1))"
done
done
