cd "$(dirname "$0")/../.."
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; tail -3 gpurun_out/pytest_gpu4.log
python tools/stage_bench.py c2 c3 2>&1 | grep "^c"
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-large 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['value'],1), d['gpu_launches'] if 'gpu_launches' in d else '')"; done
