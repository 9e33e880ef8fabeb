#!/usr/bin/env python
"""Warp-stall samples per CUDA source line of one kernel in an ncu report.

usage: python tools/ncu_lines.py REPORT LAUNCH_INDEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx),
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
fname, total, per = None, 0, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] and len(r) > 4 and r[4].isdigit():  # a source line row
        n = int(r[4])
        total += n
        per[(fname, int(r[0]), r[1].strip()[:70])] = per.get((fname, int(r[0]), r[1].strip()[:70]), 0) + n
print("samples", total)
for (f, ln, src), n in sorted(per.items(), key=lambda x: -x[1])[:top]:
    print(f"{n * 100 / max(total, 1):5.1f}%  {f}:{ln}  {src}")
