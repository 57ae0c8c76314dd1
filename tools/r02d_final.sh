#!/bin/bash
# round-2 final evidence (batch 4): GPU suite, memcheck, bench lines of every config + reference arm,
# ncu launch list of the bench command, full-set K1 / K2 / K3 captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_small.py > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
for c in hurricane hacc hacc_ridges; do
  timeout 600 python bench.py --config $c --sweep "" > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
done
timeout 600 python bench.py --config cesm > gpurun_out/r02_bench_cesm.json 2> gpurun_out/r02_bench_cesm.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --kernel-reps 2 --e2e-steps 1 --no-cpu --sweep "" > gpurun_out/bench_under_ncu.log 2>&1
for k in compress128 decode128 index128; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 -o gpurun_out/r02_${k} python tools/kernel_times.py > gpurun_out/ncu_${k}.log 2>&1
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
python tools/generic_times.py 64 128 256 512 > gpurun_out/r02_block_sizes.txt 2>&1
timeout 300 python tools/e2e_pipeline.py 8 16 > gpurun_out/r02_e2e_pipeline.txt 2>&1
