#!/usr/bin/env python
"""Hot SASS instructions of one kernel in an ncu report (warp-stall samples).

usage: python tools/ncu_hot.py REPORT LAUNCH_INDEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx),
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [(k, r[isrc], int(r[iss] or 0)) for k, r in enumerate(rows[1:])
        if len(r) > iss and (r[iss] or "0").isdigit()]
total = sum(d[2] for d in data)
print(lines[0][:160])
print("instructions", len(data), "samples", total)
ops = {}
for _, s, n in data:
    op = s.split()[0] if s.split() else "?"
    if op.startswith("@"):
        op = s.split()[1]
    op = op.split(".")[0]
    ops[op] = ops.get(op, 0) + n
print("by opcode:", ", ".join(f"{k}={v * 100 / total:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:14]))
for k, s, n in sorted(data, key=lambda x: -x[2])[:top]:
    print(f"{k:5d} {n * 100 / total:5.1f}%  {s}")
