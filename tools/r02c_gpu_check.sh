#!/bin/bash
# round-2 session-3 GPU check at HEAD: suite, bench, K1 variant A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
K1_VARIANTS=1,2,3 timeout 600 python tools/k1_ab.py nyx1e-3 nyx1e-2 nyx1e-4 hurricane hacc noise > gpurun_out/k1_ab.json 2>&1
