#!/bin/bash
# DRAM traffic per stage kernel for every config (live states) -> profiles/ncu_traffic_r02.json
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python tools/traffic_capture.py c0 c1 c2 c3 c4 > gpurun_out/traffic_plain_r02d.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/traffic_plain_r02d.log
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum \
    --clock-control none --csv --log-file gpurun_out/traffic_r02d.csv \
    python tools/traffic_capture.py c0 c1 c2 c3 c4 > gpurun_out/traffic_capture_r02d.log 2>&1; echo "ncu rc=$?"
