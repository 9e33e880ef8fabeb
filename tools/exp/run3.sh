cd "$(dirname "$0")/../.."
python -m pytest tests/test_gpu_kernels.py -q -x -k "ponly or bulk or ring_tma or split" 2>&1 | tail -2
unset SDCSW_LIB_PATH; python tools/exp/gemm_knobs.py kq8 2>&1 | grep -v Warning
python tools/stage_bench.py c3 2>&1 | grep "^c"
