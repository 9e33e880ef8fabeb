#!/bin/bash
# first inverse ring pass: staged in shared memory (base) vs loaded straight from the Fourier
# workspace (p0d, SDCSW_RING_P0DIRECT=1); ring stage times, step times, f_E bitwise
cd "$(dirname "$0")/../.."
for r in 1 2; do
for v in p0d base; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python tools/exp/ring_ab2.py $v 63:1,3 127:1,4,256 255:4 511:5 2>&1 | grep ring
  python tools/exp/cfg_time.py c0 c1 c2 2>&1 | grep "^c" | sed "s/^/$v /"
done
done
python -c "
import numpy as np
for T in (63, 127, 255, 511):
    a=np.load(f'gpurun_out/ab/fe_base_{T}.npy'); b=np.load(f'gpurun_out/ab/fe_p0d_{T}.npy')
    print(T, 'staged == direct bitwise:', np.array_equal(a.view(np.uint64), b.view(np.uint64)))
"
