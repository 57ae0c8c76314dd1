#!/bin/bash
mkdir -p gpurun_out
unset SZX_NVCC_FLAGS
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -q -x > gpurun_out/vpl_parity.log 2>&1
echo "rc=$?" >> gpurun_out/vpl_parity.log
bash tools/k2_knobs.sh "" "-DSZX_K2_VPL=16" > gpurun_out/vpl_knobs.txt 2>&1
