#!/usr/bin/env python
"""Per-CUDA-source-line instruction counts and stall samples from an ncu report (run here).

    tools/ncu_lines.py X.ncu-rep [--top 50]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=50):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    f = None
    agg = {}
    hdr = None
    for r in csv.reader(io.StringIO(txt)):
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 8 or not r[0]:
            continue
        # ncu does not escape quotes inside source text: index metric columns from the right
        def col(name):
            return r[len(r) - (len(hdr) - hdr.index(name))]
        try:
            inst = int(col("Instructions Executed") or 0)
            st = int(col("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            continue
        k = (f, int(r[0]))
        a = agg.setdefault(k, [0, 0, r[1][:100]])
        a[0] += inst
        a[1] += st
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-inst {ti}, stall samples {ts}")
    for (f, ln), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * i / ti:5.1f}% inst {i:>11d} stall {100 * s / ts:5.1f}%  {f}:{ln:<4d} {src.strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 50)
