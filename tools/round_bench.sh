#!/bin/bash
# One GPU call: default bench (driver flags) + reference arm + ncu DRAM traffic
# of the stage kernels (c1, c3) for profiles/ncu_traffic_r02.json.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${TAG:-r02}
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_${tag}.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${tag}_reference.json 2> gpurun_out/bench_${tag}_ref.err; echo "ref rc=$?"
if [ "${TRAFFIC:-1}" = 1 ]; then
  python tools/traffic_capture.py c1 c3 > gpurun_out/traffic_capture_plain.log 2>&1 && \
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic_${tag}.csv \
      python tools/traffic_capture.py c1 c3 > gpurun_out/traffic_capture.log 2>&1; echo "ncu rc=$?"
fi
