#!/bin/bash
# ncu --set full (source counters) of K1 v1 and v3 on NYX 1e-3
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"compress128" -s 3 -c 1 -o gpurun_out/k1v1_nyx python tools/k1_probe.py 1 > gpurun_out/ncu1.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"compress128" -s 3 -c 1 -o gpurun_out/k1v3_nyx python tools/k1_probe.py 3 > gpurun_out/ncu3.log 2>&1
