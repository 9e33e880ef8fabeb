# dSDC step rate with the table-streaming (bulk) analysis forced on at smaller truncations
for c in c2 c1 c0; do
  python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c default', round(d['value'],1), d['config']['stage_us']['legendre_analysis'])"
  SDCSW_TMA_MIN_T=60 SDCSW_ANAL_WJ=4 python bench.py --config $c --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c tma', round(d['value'],1), d['config']['stage_us']['legendre_analysis'])"
done
