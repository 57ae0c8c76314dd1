#!/usr/bin/env python
"""Exact per-source-line instruction counts from an ncu report: every SASS instruction counted
once (ncu's cuda,sass view lists an inlined instruction under several source lines; here each
address goes to the LAST source line it is listed under -- the innermost one).

    tools/ncu_sass_lines.py X.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    owner = {}
    cur = None
    f = None
    hdr = None
    src = {}
    for r in csv.reader(io.StringIO(txt)):
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 4:
            continue
        if r[0]:
            cur = (f, int(r[0]))
            src[cur] = r[1][:90]
        elif r[2].startswith("0x") and cur:
            owner[r[2]] = cur  # last listing wins
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                           "sass"], capture_output=True, text=True).stdout
    cnt = collections.Counter()
    tot = 0
    h = None
    for r in csv.reader(io.StringIO(sass)):
        if r and r[0] == "Address":
            h = r
            continue
        if h and r and r[0].startswith("0x"):
            c = int(r[h.index("Instructions Executed")] or 0)
            tot += c
            cnt[owner.get(r[0], ("?", 0))] += c
    print(f"total warp-inst {tot}")
    for (fl, ln), c in cnt.most_common(top):
        print(f"{100 * c / tot:5.1f}% {c:>11d}  {fl}:{ln:<5d} {src.get((fl, ln), '').strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
