#!/bin/bash
cd "$(dirname "$0")/../.."
for r in 1 2; do
for v in noprune base; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python tools/exp/ring_ab2.py $v 127:1,4,256 511:1,5 255:4 2>&1 | grep ring
  python tools/stage_bench.py c1 2>&1 | grep "^c" | sed "s/^/$v /"
done
done
python -c "
import numpy as np
for T in (127, 255, 511):
    a=np.load(f'gpurun_out/ab/fe_base_{T}.npy'); b=np.load(f'gpurun_out/ab/fe_noprune_{T}.npy')
    print(T, 'pruned == unpruned bitwise:', np.array_equal(a.view(np.uint64), b.view(np.uint64)))
"
