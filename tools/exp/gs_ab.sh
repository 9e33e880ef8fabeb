#!/bin/bash
# steps per replayed CUDA graph (c1 bench value)
cd "$(dirname "$0")/../.."
for r in 1 2; do
for g in 8 25 50; do
  SDCSW_GRAPH_STEPS=$g python bench.py --steps 10 --warmup 3 --no-cpu --no-large 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gs$g c1', round(d['value'],1))"
done
done
