# analysis stage time vs states per CTA (SDCSW_ANA_NB)
for v in 0 1 2 3; do
  SDCSW_ANA_NB=$v python - <<PY
import sys; sys.path.insert(0, '.')
from bench import time_stage
from paper_2403_20135_b200.problem import SphericalShallowWater
for T in (255, 511):
    p = SphericalShallowWater(T, device=0, max_batch=5)
    for nb in ((1, 4, 5) if T > 400 else (1, 4)):
        print("ana_nb=$v", T, nb, "analysis %.1f us" % (time_stage(p, 2, nb, reps=20) * 1e6), flush=True)
    p.close()
PY
done
