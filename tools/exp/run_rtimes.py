import ctypes, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2403_20135_b200 import _native
import os
_native.LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), 'build/var/exp4.so')
L = _native.load(_native.LIB_PATH)
import bench, torch
from paper_2403_20135_b200.problem import SphericalShallowWater
runs = [(a.split(':')[0], int(a.split(':')[1])) for a in sys.argv[1:]] or [('c1', 1), ('c1', 4)]
for cfg, nb in runs:
    c = bench.CONFIGS[cfg]
    p = SphericalShallowWater(c['trunc'], max_batch=max(nb, 4))
    bench.time_stage(p, 0, nb, reps=3)
    u = p.empty_states(nb); out = p.empty_states(nb)
    for _ in range(3):
        L.sdcsw_transform_stage(p.handle, 1, u.data_ptr(), out.data_ptr(), nb, p.stream())
    os.environ.get('X')
    torch.cuda.synchronize()
    n = min(p.grid.nlat // 2 * nb, 8192)
    buf = (ctypes.c_ulonglong * (8 * n))()
    L.sdcsw_debug_rtimes.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.sdcsw_debug_rtimes(buf, 8 * n)
    t = np.array(buf, dtype=np.float64).reshape(n, 8)
    t = t[:, [0, 6, 7, 1, 2, 3, 4, 5]]
    d = np.diff(t, axis=1)  # SM cycles per phase
    print(cfg, nb, 'cycles per phase (twiddles, wait+input, pass0, inv, prod, fwd, out): mean',
          np.round(d.mean(0)), 'max', np.round(d.max(0)), 'total mean', round(d.sum(1).mean()), flush=True)
