#!/bin/bash
cd "$(dirname "$0")/../.."
for r in 1 2; do
for v in notw base; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python tools/exp/ring_ab2.py $v 63:1,3 127:1,4,256 255:4 511:5 2>&1 | grep ring
  python tools/stage_bench.py c0 c1 2>&1 | grep "^c" | awk -v f=$v '{print f, $1, $(NF-1), $NF}'
done
done
python -c "
import numpy as np
for T in (63, 127, 255, 511):
    a=np.load(f'gpurun_out/ab/fe_base_{T}.npy'); b=np.load(f'gpurun_out/ab/fe_notw_{T}.npy')
    print(T, 'tw-all vs branch bitwise:', np.array_equal(a.view(np.uint64), b.view(np.uint64)))
"
