#!/bin/bash
mkdir -p gpurun_out
unset SZX_NVCC_FLAGS
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "TestCompressVariants or TestRingPaths or TestWarpPaths or golden or multi" > gpurun_out/mbx_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/mbx_pytest.log
bash tools/k1_knobs.sh "" "-DSZX_K1_STATIC=1" "-DSZX_K1_MBX=0" > gpurun_out/mbx_knobs.txt 2>&1
