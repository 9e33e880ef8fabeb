# ring stage time per variant: VARS="base twg ..." TS="511"
for v in ${VARS:-base}; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  python - <<PY
import sys; sys.path.insert(0, '.')
from bench import time_stage
from paper_2403_20135_b200.problem import SphericalShallowWater
for T in [int(x) for x in "${TS:-511}".split()]:
    p = SphericalShallowWater(T, device=0, max_batch=5)
    for nb in ((1, 4, 5) if T > 200 else (1, 4)):
        print("$v", T, nb, "ring %.1f us" % (time_stage(p, 1, nb, reps=20) * 1e6), flush=True)
    p.close()
PY
done
