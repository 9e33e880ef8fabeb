#!/bin/bash
# GPU test pass + memcheck of the bulk-synthesis partial-block shapes (one sanitizer tool).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
if [ "${MEMCHECK:-0}" = 1 ]; then
  timeout 600 compute-sanitizer --tool memcheck python tools/exp/memcheck_synb.py > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.log
  tail -5 gpurun_out/memcheck.log
fi
