#!/bin/bash
# round-2 GPU check: full GPU suite with durations, memcheck, K0 timing + ncu, host info
mkdir -p gpurun_out
(free -g; nproc; nvidia-smi --query-gpu=name,memory.total --format=csv) > gpurun_out/host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_small.py > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/memcheck.log
python tools/k0_probe.py > gpurun_out/k0.json 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:range -s 3 -c 1 -o gpurun_out/k0 python tools/k0_probe.py > gpurun_out/k0_ncu.log 2>&1
