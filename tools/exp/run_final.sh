#!/bin/bash
# Bench lines of every config (c1 in the driver's format with its reference arm; c0, c2, c3, c4
# with CPU baselines) -> gpurun_out/bench_${TAG}_*.json
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
tag=${TAG:-r02_v3}
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${tag}_c1.json 2> gpurun_out/bench_${tag}_c1.err; echo "c1 rc=$?"
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${tag}_c1_reference.json 2> gpurun_out/bench_${tag}_c1_ref.err; echo "ref rc=$?"
for c in c0 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-large > gpurun_out/bench_${tag}_${c}.json 2> gpurun_out/bench_${tag}_${c}.err
  echo "$c rc=$?"
done
for f in gpurun_out/bench_${tag}_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d.get('value',0),1), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'))"; done
