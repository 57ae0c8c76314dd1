#!/usr/bin/env python
"""Summarise ncu artefacts for profiles/ (run here, on the CPU box).

  tools/ncu_summary.py report X.ncu-rep [--top 25]   key metrics + hottest SASS (stall samples)
  tools/ncu_summary.py launches launches.csv          per-kernel launch times (szx kernels)
  tools/ncu_summary.py traffic X.ncu-rep              dram read+write bytes per launch (JSON)
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "lts__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw_rows(rep):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    head, units, data = rows[0], rows[1], rows[2:]
    return head, units, data


def report(rep, top=25):
    head, units, data = raw_rows(rep)
    out = []
    for row in data:
        name = row[head.index("Kernel Name")]
        out.append(f"kernel: {name}")
        for k in KEYS:
            if k in head:
                i = head.index(k)
                out.append(f"  {k:70s} {row[i]:>16s} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv",
                                           "--print-source", "sass"]))))
    h = src[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    ii = h.index("Instructions Executed")
    items = []
    for k, r in enumerate(src[2:]):
        try:
            items.append((int(r[si] or 0), int(r[ii] or 0), k, r[1].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(x[0] for x in items) or 1
    toti = sum(x[1] for x in items)
    out.append(f"  SASS instructions: {len(items)}, warp-instructions executed: {toti}, "
               f"stall samples: {tot}")
    out.append("  hottest SASS by stall samples:")
    for s, i, k, txt in sorted(items, reverse=True)[:top]:
        out.append(f"    {100 * s / tot:5.1f}%  inst={i:>10d}  #{k:<5d} {txt[:80]}")
    return "\n".join(out)


def launches(path):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if not ln.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    acc = {}
    for r in rows[1:]:
        if "szx::" not in r[ki]:
            continue
        name = r[ki].split("(")[0]
        acc.setdefault(name, []).append(float(r[vi].replace(",", "")))
    out = []
    tot = sum(sum(v) for v in acc.values())
    for name, v in acc.items():
        out.append(f"{name:40s} launches={len(v):4d} mean={sum(v) / len(v) / 1e3:9.2f} us "
                   f"share={100 * sum(v) / tot:5.1f}%")
    return "\n".join(out)


def traffic(rep):
    head, units, data = raw_rows(rep)
    res = {}
    for row in data:
        name = row[head.index("Kernel Name")].split("(")[0]
        def val(k):
            v = float(row[head.index(k)].replace(",", ""))
            u = units[head.index(k)]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        res[name] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    return json.dumps(res)


if __name__ == "__main__":
    cmd, path = sys.argv[1], sys.argv[2]
    print({"report": report, "launches": launches, "traffic": traffic}[cmd](path))
