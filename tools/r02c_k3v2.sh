#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "TestIndexKernels or TestK1Index" > gpurun_out/k3v2_pytest.log 2>&1
echo "k3v2 rc=$?" >> gpurun_out/k3v2_pytest.log
python tools/kernel_times.py > gpurun_out/k3v2_kt.txt 2>&1
python tools/kernel_times.py 25000000 >> gpurun_out/k3v2_kt.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
