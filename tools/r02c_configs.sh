#!/bin/bash
# r02: bench line of every BASELINE config (headline NYX is profiles/r02_bench.json)
mkdir -p gpurun_out
for c in hurricane hacc hacc_ridges; do
  timeout 600 python bench.py --config $c --sweep "" > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
done
timeout 600 python bench.py --config cesm > gpurun_out/r02_bench_cesm.json 2> gpurun_out/r02_bench_cesm.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
