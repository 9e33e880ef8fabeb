#!/usr/bin/env python
"""Stage roofline fractions as the bench line reports them: the c3 (T511) block's stage
kernels (live states; node kernels with L2 flushed per launch) and the c1 stage times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

blk = bench.large_truncation_block("c3", n_steps=10)
print(f"c3 steps/s {blk['steps_per_s']:.1f}")
for name, d in blk["stages"].items():
    for nb, r in d.items():
        print(f"c3 {name:20s} {nb:4s} {r['us_per_launch']:8.1f} us  frac {r['frac']:.3f} ({r['unit']})")
