#!/bin/bash
# K1 v1 static tile assignment: parity, A/B vs dynamic claiming, per-tile trace
mkdir -p gpurun_out
unset SZX_NVCC_FLAGS
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "TestCompressVariants or TestRingPaths or TestWarpPaths or golden" > gpurun_out/static_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/static_pytest.log
K1_VARIANTS=1 timeout 200 python tools/k1_ab.py nyx1e-3 nyx1e-4 hurricane hacc noise > gpurun_out/static_ab.json 2>&1
export SZX_NVCC_FLAGS="-DSZX_K1_STATIC=0"
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
K1_VARIANTS=1 timeout 200 python tools/k1_ab.py nyx1e-3 nyx1e-4 hurricane hacc noise > gpurun_out/dynamic_ab.json 2>&1
export SZX_NVCC_FLAGS="-DSZX_TRACE"
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
python tools/k1_trace.py > gpurun_out/k1_trace_static.txt 2>&1; python tools/k1_trace.py random_walk 280953867 >> gpurun_out/k1_trace_static.txt 2>&1
