#!/bin/bash
cd "$(dirname "$0")/../.."
for r in 1 2; do
for wj in 2 3; do
  SDCSW_SYNP_WJ=$wj python tools/exp/gemm_knobs.py wj$wj 2>&1 | grep T127
  SDCSW_SYNP_WJ=$wj timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-large 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('wj$wj c4', round(d['value'],1))"
done
done
