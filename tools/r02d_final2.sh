# after the batched decode index: GPU suite, smoke, NYX + CESM bench lines
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 600 python bench.py --config cesm > gpurun_out/r02_bench_cesm.json 2> gpurun_out/r02_bench_cesm.err
