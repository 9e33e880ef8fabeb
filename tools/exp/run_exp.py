import os, sys, shutil
sys.path.insert(0, '/root/repo')
from paper_2403_20135_b200 import _native
v = sys.argv[1]
if v != '0':
    _native.LIB_PATH = f'/root/repo/tools/exp/libsdcsw_exp{v}.so'
    _native.load(_native.LIB_PATH)
import bench, torch
from paper_2403_20135_b200.problem import SphericalShallowWater
for cfg in ('c0', 'c1'):
    c = bench.CONFIGS[cfg]
    p = SphericalShallowWater(c['trunc'], max_batch=4)
    for nb in (1, 4):
        bench.time_stage(p, 0, nb, reps=3)
        print(v, cfg, nb, 'synth-only %.1f' % (bench.time_stage(p, 3, nb) * 1e6))
