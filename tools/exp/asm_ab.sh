#!/bin/bash
# fused assembly (last analysis CTA per m) vs the separate assembly kernel
cd "$(dirname "$0")/../.."
python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "ponly or spectral_split or ring_tma" 2>&1 | tail -2
for r in 1 2; do
for f in 0 1; do
  SDCSW_ASM_FUSED=$f python tools/exp/gemm_knobs.py asm$f 2>&1 | grep -v Warn
  SDCSW_ASM_FUSED=$f python tools/stage_bench.py c3 2>&1 | grep "^c" | awk -v f=$f '{print "asm" f, $1, $(NF-1), $NF}'
  SDCSW_ASM_FUSED=$f timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-large 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('asm$f c4', round(d['value'],1))"
done
done
