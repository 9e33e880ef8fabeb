#!/bin/bash
# What the driver runs at round end, in its order: GPU tests, smoke, the reference arm, the bench.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
t0=$(date +%s); python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - t0 ))s"

tail -c 400 gpurun_out/final_bench.json
