#!/bin/bash
# r02 ncu captures: launch list of the bench command, full-set K1 / K2 / K3 on NYX 1e-3
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --kernel-reps 2 --e2e-steps 1 --no-cpu --sweep "" > gpurun_out/bench_under_ncu.log 2>&1
for k in compress128 decode128 index128; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 -o gpurun_out/r02_${k} python tools/kernel_times.py > gpurun_out/ncu_${k}.log 2>&1
done
