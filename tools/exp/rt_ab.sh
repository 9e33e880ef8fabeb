#!/bin/bash
cd "$(dirname "$0")/../.."
for r in 1 2 3; do
for v in base ${VARS:-rt192 rt128}; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python tools/stage_bench.py c1 2>&1 | grep "^c" | sed "s/^/$v /"
done
done
