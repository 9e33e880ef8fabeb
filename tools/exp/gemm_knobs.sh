#!/bin/bash
cd "$(dirname "$0")/../.."
for r in 1 2; do
for v in base ${VARS:-k1 k2 k3 k4 k5 k6}; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python tools/exp/gemm_knobs.py $v 2>&1 | grep -v Warning
done
done
