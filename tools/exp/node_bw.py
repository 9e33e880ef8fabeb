"""Achieved HBM bandwidth of the sweep-node and final-node kernels at T511 (M = 5)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_20135_b200 import CollocationTable, SdcConfig, SweepMode  # noqa: E402
from paper_2403_20135_b200.integrators import diagonal_step_coefficients  # noqa: E402
from paper_2403_20135_b200.parallel_nodes import CudaNodeBackend  # noqa: E402
from paper_2403_20135_b200.problem import SphericalShallowWater  # noqa: E402

T, M = 511, 5
p = SphericalShallowWater(T, max_batch=M)
cfg = SdcConfig(table=CollocationTable.radau_right(M), n_sweeps=5, mode=SweepMode.DIAGONAL_PARALLEL)
coef = diagonal_step_coefficients(cfg, 30.0, p.mean_geopotential)
blk = M * (M + 4)
b = CudaNodeBackend(p)
S = p.state_size
u0 = p.empty_states(1).normal_() if False else torch.randn(S, dtype=torch.complex128, device=p.device) * 1e-6
fe = torch.randn(M, S, dtype=torch.complex128, device=p.device) * 1e-6
fi = torch.randn(M, S, dtype=torch.complex128, device=p.device) * 1e-6
uo = p.empty_states(M)
fo = p.empty_states(M)
out = p.empty_states(1)
sc = np.ascontiguousarray(coef[:blk])
fc = np.ascontiguousarray(coef[(5 - 1) * blk:])


def tm(fn, n=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / n


sbytes = S * 16
t = tm(lambda: b.final_node(M, fc, u0, fe, 1, fi, 1, False, out))
print(f"final node: {t*1e6:.1f} us, {(2*M+2)*sbytes/1e6:.0f} MB -> {(2*M+2)*sbytes/t/1e9:.0f} GB/s")
t = tm(lambda: b.sweep_nodes(M, 0, M, sc, u0, fe, 1, fi, 1, False, uo, fo))
nb = (1 + 2 * M) * sbytes + 2 * M * sbytes
print(f"sweep nodes (u_out + fi_out): {t*1e6:.1f} us, {nb/1e6:.0f} MB -> {nb/t/1e9:.0f} GB/s")
