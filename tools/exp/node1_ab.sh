#!/bin/bash
# H-free node kernel: one thread per coefficient (all nodes) vs per (coefficient, node)
cd "$(dirname "$0")/../.."
python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.problem import SphericalShallowWater
import subprocess
PY
for r in 1 2; do
for v in 0 1; do
  SDCSW_NODE1=$v python tools/stage_bench.py c2 c3 2>&1 | grep "^c" | awk -v f=$v '{print "node1=" f, $1, $(NF-1), $NF}'
  SDCSW_NODE1=$v timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-large 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('node1=$v c4', round(d['value'],1))"
done
done
for v in 0 1; do SDCSW_NODE1=$v python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode, random_initial_state
from paper_2403_20135_b200.integrators import DeviceStepper
from paper_2403_20135_b200.problem import SphericalShallowWater
for T,M,E in ((255,4,1),(127,4,6)):
    p = SphericalShallowWater(T, max_batch=M*E)
    cfg = SdcConfig(table=CollocationTable.radau_right(M), n_sweeps=3, mode=SweepMode.DIAGONAL_PARALLEL)
    st = DeviceStepper(p, cfg, 60.0, serial=False, members=E)
    u = torch.from_numpy(np.stack([random_initial_state(p.grid, 9+e) for e in range(E)])).to(0).reshape(-1).contiguous()
    st.run(u, 3); torch.cuda.synchronize()
    np.save(f'gpurun_out/n1_{T}_$v.npy', u.cpu().numpy())
"; done
python -c "
import numpy as np
for T in (255,127):
    a=np.load(f'gpurun_out/n1_{T}_0.npy'); b=np.load(f'gpurun_out/n1_{T}_1.npy')
    print('T',T,'per-node == per-coefficient bitwise:', np.array_equal(a.view(np.uint64), b.view(np.uint64)))
"
