import sys
sys.path.insert(0, '/root/repo')
import bench
from paper_2403_20135_b200.problem import SphericalShallowWater
for name in sys.argv[1:]:
    c = bench.CONFIGS[name]
    p = SphericalShallowWater(c["trunc"], max_batch=c["nodes"])
    r = {}
    for stage, nm in ((1, "ring"), (2, "anal"), (4, "fused")):
        for nb in (1, c["nodes"]):
            bench.time_stage(p, 0, nb, reps=2)
            r[f"{nm}{nb}"] = round(bench.time_stage(p, stage, nb, reps=30) * 1e6, 1)
    print(name, r, flush=True)
