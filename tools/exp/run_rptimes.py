"""Phase cycles of item 2 of every CTA of the persistent ring kernel (SDCSW_EXP=4 build):
python tools/exp/run_rptimes.py c3:5"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from paper_2403_20135_b200 import _native  # noqa: E402
_native.LIB_PATH = os.path.join(ROOT, 'build/var/exp4.so')
L = _native.load(_native.LIB_PATH)
os.environ['SDCSW_RINGP'] = '1'
import bench, torch  # noqa: E402,E401
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402
for a in sys.argv[1:] or ['c3:5']:
    cfg, nb = a.split(':')[0], int(a.split(':')[1])
    c = bench.CONFIGS[cfg]
    p = SphericalShallowWater(c['trunc'], max_batch=nb)
    bench.time_stage(p, 0, nb, reps=3)
    u = p.empty_states(nb); out = p.empty_states(nb)
    for _ in range(3):
        L.sdcsw_transform_stage(p.handle, 1, u.data_ptr(), out.data_ptr(), nb, p.stream())
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (8 * 148))()
    L.sdcsw_debug_rtimes.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.sdcsw_debug_rtimes(buf, 8 * 148)
    t = np.array(buf, dtype=np.float64).reshape(148, 8)[:, [0, 6, 7, 1, 2, 3, 4]]
    d = np.diff(t, axis=1)
    print(cfg, nb, 'item-2 cycles (wait stage, pass0, inv, prod, fwd, out): mean', np.round(d.mean(0)),
          'max', np.round(d.max(0)), 'total', round(d.sum(1).mean()), flush=True)
