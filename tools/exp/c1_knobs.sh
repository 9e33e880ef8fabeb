#!/bin/bash
# c1/c0 step time under the plan knobs that change the latency-regime GEMM shapes
# (same box, two rounds; sha = state checksum after the run, equal sha = bitwise equal)
cd "$(dirname "$0")/../.."
for r in 1 2; do
  for knobs in "" "SDCSW_SYNTH_WJ=2" "SDCSW_ANAL_WJ=2" "SDCSW_SYN_CP=1" \
               "SDCSW_SYNTH_WJ=2 SDCSW_SYN_CP=1" "SDCSW_SYNTH_WJ=2 SDCSW_ANAL_WJ=2"; do
    echo "== r$r [$knobs]"
    env $knobs timeout 300 python tools/exp/cfg_time.py c1 c0 2>&1 | grep -E "^c[0-9]|Error" | sed "s/^/  /"
  done
done
