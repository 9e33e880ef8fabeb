#!/bin/bash
# node kernels: HEAD build (nodes_old) vs the working tree, c2/c3 steps, c4 bench value, node_bw
cd "$(dirname "$0")/../.."
for r in 1 2; do
for v in nodes_old new; do
  if [ $v = new ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python tools/stage_bench.py c2 c3 2>&1 | grep "^c" | sed "s/^/$v /" | awk '{print $1, $2, $(NF-1), $NF}'
  timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-large 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c4', round(d['value'],1))"
done
done
