#!/bin/bash
# fused last-pass/output ring (fz) vs the same plans unfused (nofz) vs the default build (base)
cd "$(dirname "$0")/../.."
for r in 1 2; do
for v in base nofz fz; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python tools/exp/ring_ab2.py $v 127:1,4,64,256 511:1,5 2>&1 | grep -v Warning
  python tools/stage_bench.py c1 c3 2>&1 | grep "^c" | sed "s/^/$v /"
done
done
python - <<'PY'
import numpy as np
for T in (127, 511):
    a = np.load(f"gpurun_out/ab/fe_fz_{T}.npy"); b = np.load(f"gpurun_out/ab/fe_nofz_{T}.npy"); c = np.load(f"gpurun_out/ab/fe_base_{T}.npy")
    print(T, "fz == nofz bitwise:", np.array_equal(a.view(np.uint64), b.view(np.uint64)),
          "fz vs base rel:", np.linalg.norm(a - c) / np.linalg.norm(c))
PY
