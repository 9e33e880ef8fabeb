#!/bin/bash
# VARS="base v1 v2" SPECS="511:1,5 255:1,4" bash tools/exp/ring_ab2.sh
cd "$(dirname "$0")/../.."
for r in 1 2; do
for v in ${VARS:-base}; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python tools/exp/ring_ab2.py $v ${SPECS:-511:1,5 255:1,4} 2>&1 | grep -v Warning
done
done
