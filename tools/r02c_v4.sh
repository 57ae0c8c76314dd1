#!/bin/bash
# K1 v4 first run: variant parity tests, A/B timing vs v1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "TestCompressVariants and 4" > gpurun_out/v4_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/v4_pytest.log
K1_VARIANTS=1,4 timeout 300 python tools/k1_ab.py nyx1e-3 nyx1e-2 nyx1e-4 hurricane hacc noise > gpurun_out/v4_ab.json 2>&1
echo "ab rc=$?" >> gpurun_out/v4_ab.json
