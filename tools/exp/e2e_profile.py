"""Host-side profile of integrate() at c1 (where the e2e line's time beyond the device time goes)."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2403_20135_b200 import (CollocationTable, DiagonalSdcStepper, SdcConfig, SweepMode,
                                   integrate, random_initial_state)
from paper_2403_20135_b200.problem import SphericalShallowWater

p = SphericalShallowWater(127, max_batch=4)
u0 = random_initial_state(p.grid, 1)
cfg = SdcConfig(table=CollocationTable.radau_right(4), n_sweeps=4, mode=SweepMode.DIAGONAL_PARALLEL)
for _ in range(3):
    integrate(p, u0, 90.0, 200, DiagonalSdcStepper(cfg))
t0 = time.perf_counter()
for _ in range(10):
    integrate(p, u0, 90.0, 200, DiagonalSdcStepper(cfg))
print("ms per run", (time.perf_counter() - t0) * 100)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    integrate(p, u0, 90.0, 200, DiagonalSdcStepper(cfg))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
