import ctypes, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2403_20135_b200 import _native
_native.LIB_PATH = '/root/repo/tools/exp/libsdcsw_exp3.so'
L = _native.load(_native.LIB_PATH)
import bench, torch
from paper_2403_20135_b200.problem import SphericalShallowWater
c = bench.CONFIGS['c1']
p = SphericalShallowWater(c['trunc'], max_batch=4)
nb = 4
bench.time_stage(p, 0, nb, reps=3)
u = p.empty_states(nb); out = p.empty_states(nb)
for _ in range(3):
    L.sdcsw_transform_stage(p.handle, 3, u.data_ptr(), out.data_ptr(), nb, p.stream())
torch.cuda.synchronize()
n = 768
buf = (ctypes.c_ulonglong * (8 * n))()
L.sdcsw_debug_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.sdcsw_debug_times(buf, 8 * n)
t = np.array(buf, dtype=np.float64).reshape(n, 8)
t0 = t[:, 0].min()
st, lp, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
print('span us', en.max(), 'start range', st.min(), st.max())
print('loop dur us: mean %.2f max %.2f; epilogue mean %.2f max %.2f' % ((lp - st).mean(), (lp - st).max(), (en - lp).mean(), (en - lp).max()))
gx = 6
for m in (0, 1, 32, 64, 127):
    ids = [m * gx + x for x in range(gx)]
    print('m', m, 'start', np.round(st[ids], 2), 'loop', np.round((lp - st)[ids], 2), 'epi', np.round((en - lp)[ids], 2))
sm = t[:, 3].astype(int)
print('CTAs per SM max', np.bincount(sm).max(), 'SMs used', len(np.unique(sm)))

pro, f1, kl = (t[:, 4] - t0) / 1e3, (t[:, 5] - t0) / 1e3, (t[:, 6] - t0) / 1e3
for m in (0, 64, 127):
    i = m * gx
    print('m', m, 'start %.2f prologue %.2f firstfetch %.2f kloop %.2f reduce %.2f end %.2f' % (st[i], pro[i], f1[i], kl[i], lp[i], en[i]))
