#!/bin/bash
mkdir -p gpurun_out
unset SZX_NVCC_FLAGS
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pipe_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pipe_parity.log
timeout 300 python tools/stress_k1.py 30 >> gpurun_out/pipe_parity.log 2>&1
bash tools/k1_knobs.sh "" "-DSZX_K1_PIPE=0" "" "-DSZX_K1_PIPE=0" > gpurun_out/pipe_knobs.txt 2>&1
