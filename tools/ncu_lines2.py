#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples from an ncu report (CPU box):

    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv
    tools/ncu_lines2.py X.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
files = []
i = 0
agg = defaultdict(lambda: [0, 0, ""])
cur_file = ""
hdr = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:
        line = (cur_file, r[0], r[1][:90])
    if line is None or len(r) <= ie:
        continue
    try:
        n = int(r[ie] or 0)
        s = int(r[ss] or 0)
    except ValueError:
        continue
    a = agg[line[:2]]
    a[0] += n
    a[1] += s
    a[2] = line[2]
tot = sum(v[0] for v in agg.values())
stot = sum(v[1] for v in agg.values())
print(f"total warp instructions {tot}, stall samples {stot}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:>11} {100 * v[0] / tot:5.1f}%  stall {100 * v[1] / max(stot, 1):5.1f}%  {k[0]}:{k[1]}  {v[2].strip()}")
