#!/bin/bash
# node kernels' CTA size (SDCSW_NODE_THREADS) on the c3 block's stage fractions and the step
cd "$(dirname "$0")/../.."
for r in 1 2; do
for t in 256 128 64; do
  echo "== threads $t"
  SDCSW_NODE_THREADS=$t python tools/exp/stage_fracs.py 2>&1 | grep -E "^c3|Error"
  SDCSW_NODE_THREADS=$t python tools/exp/cfg_time.py c1 c2 c4 2>&1 | grep "^c"
done
done
