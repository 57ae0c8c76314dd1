#!/usr/bin/env python
"""Stall-reason totals and the hottest SASS lines with their reasons (run here).

    tools/ncu_stalls.py X.ncu-rep [--top 15]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=15):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    # one section per profiled launch ("Kernel Name" row, header row, data): take the first
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    h, data = rows[starts[0] + 1], rows[starts[0] + 2:starts[1]]
    si = h.index("Warp Stall Sampling (All Samples)")
    stalls = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
    items = []
    for r in data:
        try:
            items.append((int(r[si] or 0), r))
        except (ValueError, IndexError):
            pass
    tot = sum(x[0] for x in items) or 1
    agg = {}
    for _, r in items:
        for i in stalls:
            try:
                agg[h[i]] = agg.get(h[i], 0) + int(r[i] or 0)
            except ValueError:
                pass
    print("stall samples", tot)
    print("  " + ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in
                           sorted(agg.items(), key=lambda x: -x[1])[:10]))
    for s, r in sorted(items, key=lambda x: -x[0])[:top]:
        reasons = sorted([(int(r[i] or 0), h[i][6:]) for i in stalls if r[i] not in ("", "-")],
                         reverse=True)[:3]
        print(f"{100 * s / tot:5.1f}%  {r[1].strip()[:60]:60s} {reasons}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 15)
