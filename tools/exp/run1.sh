cd $GRAFT_REPO_ROOT
bash tools/gpu_tests.sh
for c in c2 c3 c4; do
  for po in 0 1; do
    SDCSW_PONLY=$po timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-large > gpurun_out/b1_${c}_po$po.json 2> gpurun_out/b1_${c}_po$po.err
    echo "$c po=$po rc=$? $(python -c "import json;d=json.load(open('gpurun_out/b1_${c}_po$po.json'));print(round(d['value'],1), d['e2e']['value'] if d.get('e2e') else '')")"
  done
done
