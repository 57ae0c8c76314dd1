#!/bin/bash
mkdir -p gpurun_out
unset SZX_NVCC_FLAGS
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "TestCompressVariants and 5" > gpurun_out/v5_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/v5_pytest.log
K1_VARIANTS=1,5 timeout 300 python tools/k1_ab.py nyx1e-3 nyx1e-4 hurricane hacc noise > gpurun_out/v5_ab.json 2>&1
for f in "-DSZX_V5_SCAN=1 -DSZX_V5_WRITERS=2" "-DSZX_V5_TEAMS=1 -DSZX_V5_SCAN=1 -DSZX_V5_WRITERS=2 -DSZX_V5_IN=4 -DSZX_V5_REC=8 -DSZX_V5_RING_KB=72"; do
  export SZX_NVCC_FLAGS="$f"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== flags: $f" >> gpurun_out/v5_ab.json
  K1_VARIANTS=5 timeout 200 python tools/k1_ab.py nyx1e-3 hacc noise >> gpurun_out/v5_ab.json 2>&1
done
