cd $GRAFT_REPO_ROOT
bash tools/gpu_tests.sh
python tools/exp/ponly_check.py 127:16:16 255:4:4 511:5:1 511:5:5 > gpurun_out/ponly1.log 2>&1; tail -12 gpurun_out/ponly1.log
