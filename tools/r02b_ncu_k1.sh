#!/bin/bash
# ncu --set full of both bs==128 compress variants on NYX 1e-3, and v1 on HACC walk
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"compress128|encode128" -s 3 -c 1 -o gpurun_out/k1v1_nyx python tools/k1_probe.py 1 > gpurun_out/ncu1.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"compress128|encode128" -s 3 -c 1 -o gpurun_out/k1v2_nyx python tools/k1_probe.py 2 > gpurun_out/ncu2.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"compress128|encode128" -s 3 -c 1 -o gpurun_out/k1v1_hacc python tools/k1_probe.py 1 random_walk 280953867 > gpurun_out/ncu3.log 2>&1
