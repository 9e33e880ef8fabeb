import ctypes, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2403_20135_b200 import _native
_native.LIB_PATH = '/root/repo/tools/exp/lib_x3.so'
L = _native.load(_native.LIB_PATH)
import torch
from paper_2403_20135_b200.problem import SphericalShallowWater
p = SphericalShallowWater(127, max_batch=4)
for nb in (1, 4):
    u = p.empty_states(nb); u.zero_(); out = p.empty_states(nb); out.zero_()
    for st in (0, 1):
        L.sdcsw_transform_stage(p.handle, st, u.data_ptr(), out.data_ptr(), nb, p.stream())
    for _ in range(3):
        L.sdcsw_transform_stage(p.handle, 4, u.data_ptr(), out.data_ptr(), nb, p.stream())
    torch.cuda.synchronize()
    n = 576
    buf = (ctypes.c_longlong * (8 * n))()
    L.sdcsw_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.sdcsw_debug_phases(buf, 8 * n)
    t = np.array(buf, dtype=np.float64).reshape(n, 8)
    d = np.diff(t[:, :5], axis=1)
    print(f"nb={nb} cycles (prologue->wait, main loop, reduction, epilogue) mean", np.round(d.mean(0)), "max", np.round(d.max(0)))
    g0, g1 = t[:, 5], t[:, 6]
    print("  global span us", (g1.max() - g0.min()) / 1e3, "start spread us", (g0.max() - g0.min()) / 1e3,
          "per-CTA us mean", ((g1 - g0) / 1e3).mean(), "CTAs per SM max", np.bincount(t[:, 7].astype(int)).max())
    order = np.argsort(g0)
    late = order[-20:]
    print("  last-started CTAs start at us", np.round((g0[late] - g0.min()) / 1e3, 2)[:10])
