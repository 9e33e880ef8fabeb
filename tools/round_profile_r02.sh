#!/bin/bash
# ncu evidence for round 2: c1 launch list of the bench command, DRAM traffic per
# stage kernel (c1, c3) and one --set full capture of every stage kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${TAG:-r02}
cmd="python bench.py --steps 2 --warmup 3 --no-cpu --no-large"
$cmd > gpurun_out/plain_${tag}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 400 --csv \
    --log-file gpurun_out/launches_${tag}.csv $cmd > gpurun_out/ncu_launch_${tag}.log 2>&1; echo "launch list rc=$?"
python tools/traffic_capture.py c1 c2 c3 > gpurun_out/traffic_plain_${tag}.log 2>&1 && \
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/traffic_${tag}.csv \
    python tools/traffic_capture.py c1 c2 c3 > gpurun_out/traffic_capture_${tag}.log 2>&1; echo "traffic rc=$?"
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -o gpurun_out/prof_${tag}_stages python tools/traffic_capture.py ${FULL_CFGS:-c1 c2 c3} > gpurun_out/ncu_full_${tag}.log 2>&1; echo "full rc=$?"
