#!/bin/bash
# node kernel assembling f_E from the P analyses (nodes_asm) vs the assembly kernel
cd "$(dirname "$0")/../.."
python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "node_kernel_operand or ponly_stepper" 2>&1 | tail -2
for r in 1 2; do
for a in 0 1; do
  SDCSW_NODES_ASM=$a python tools/stage_bench.py c2 c3 2>&1 | grep "^c" | awk -v f=$a '{print "asm" f, $1, $(NF-1), $NF}'
  SDCSW_NODES_ASM=$a timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-large 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('asm$a c4', round(d['value'],1))"
done
done
