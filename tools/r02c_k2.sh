#!/bin/bash
mkdir -p gpurun_out
python tools/kernel_times.py > gpurun_out/k2_kt.txt 2>&1
python tools/kernel_times.py 280953867 >> gpurun_out/k2_kt.txt 2>&1
python tools/kernel_times.py 25000000 >> gpurun_out/k2_kt.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
