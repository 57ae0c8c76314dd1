mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "TestCompressVariants" > gpurun_out/v3_parity.log 2>&1; echo rc=$? >> gpurun_out/v3_parity.log
K1_VARIANTS=1,3 timeout 300 python tools/k1_ab.py nyx1e-3 nyx1e-2 nyx1e-4 hurricane hacc noise > gpurun_out/k1_ab3.json 2>&1
