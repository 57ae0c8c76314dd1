#!/bin/bash
mkdir -p gpurun_out
unset SZX_NVCC_FLAGS
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "TestCompressVariants or TestRingPaths or TestWarpPaths or golden or multi" > gpurun_out/lbhi_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/lbhi_pytest.log
bash tools/k1_knobs.sh "" "-DSZX_K1_FWD=8" "-DSZX_K1_STATIC=0" "-DSZX_K1_SCAN=2 -DSZX_K1_WRITERS=1" "-DSZX_K1_LBHI=0" > gpurun_out/lbhi_knobs.txt 2>&1
export SZX_NVCC_FLAGS="-DSZX_TRACE"
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
python tools/k1_trace.py > gpurun_out/k1_trace5.txt 2>&1; python tools/k1_trace.py random_walk 280953867 >> gpurun_out/k1_trace5.txt 2>&1
