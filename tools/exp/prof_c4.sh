#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_synthesis_bulk|k_analysis_bulk_ponly|k_ring|k_xsyn_ponly|k_assemble_ponly" \
    -o gpurun_out/prof_r02d_c4 python tools/traffic_capture.py c4 > gpurun_out/ncu_full_r02d_c4.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/prof_r02d_c4.ncu-rep
