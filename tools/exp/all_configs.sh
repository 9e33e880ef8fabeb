#!/bin/bash
# bench lines of c0, c2, c3, c4 (with CPU baselines) -> gpurun_out/bench_${TAG}_cN.json
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
tag=${TAG:-r02_v2}
for c in c0 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${tag}_${c}.json 2> gpurun_out/bench_${tag}_${c}.err
  echo "$c rc=$?"
done
