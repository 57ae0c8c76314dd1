#!/bin/bash
mkdir -p gpurun_out
unset SZX_NVCC_FLAGS
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "TestCompressVariants and 4" > gpurun_out/v4s_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/v4s_pytest.log
bash tools/v4_sweep.sh "5 2 1 0" "5 3 1 0" "5 2 2 0" "4 2 1 0" > gpurun_out/v4s_sweep.txt 2>&1
