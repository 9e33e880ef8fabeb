#!/bin/bash
# TMA ring output stores vs plain stores: bitwise f_E, stage times, c1/c2/c3 steps
set -x
mkdir -p gpurun_out
CASES="63:1 127:1 127:4 127:16:64 255:4 511:1 511:5 85:3 42:2"
for m in 0 1; do
  SDCSW_RING_TMA_STORE=$m timeout 600 python tools/exp/ring_store_ab.py /tmp/rs$m $CASES
done
python tools/exp/ring_store_ab.py --compare /tmp/rs0 /tmp/rs1; echo "compare exit $?"
for rep in 1 2; do
for m in 0 1; do
  for c in c1 c2; do
    SDCSW_RING_TMA_STORE=$m timeout 300 python bench.py --config $c --no-cpu --no-large --steps 200 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('store=$m $c', d['value'], d['e2e']['value'])"
  done
done
done
for m in 0 1; do
  SDCSW_RING_TMA_STORE=$m timeout 600 python bench.py --config c3 --no-cpu --no-large --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('store=$m c3', d['value'], d['e2e']['value'])"
done
