#!/bin/bash
# ncu evidence after the H-free transforms: c1 launch list of the bench command, DRAM
# traffic per stage (c1, c2, c3), and a --set full capture of the c3 H-free stage kernels
# (kept under the 64 MiB gpurun_out limit: c3 only, stage kernels only).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${TAG:-r02c}
cmd="python bench.py --steps 2 --warmup 3 --no-cpu --no-large"
$cmd > gpurun_out/plain_${tag}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 400 --csv \
    --log-file gpurun_out/launches_${tag}.csv $cmd > gpurun_out/ncu_launch_${tag}.log 2>&1; echo "launch list rc=$?"
python tools/traffic_capture.py c1 c2 c3 > gpurun_out/traffic_plain_${tag}.log 2>&1 && \
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/traffic_${tag}.csv \
    python tools/traffic_capture.py c1 c2 c3 > gpurun_out/traffic_capture_${tag}.log 2>&1; echo "traffic rc=$?"
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_synthesis_bulk|k_analysis_bulk_ponly|k_ring|k_xsyn_ponly|k_prep_ponly|k_assemble_ponly|k_sweep_nodes_po" \
    -o gpurun_out/prof_${tag}_c3 python tools/traffic_capture.py c3 > gpurun_out/ncu_full_${tag}.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/prof_${tag}_c3.ncu-rep
