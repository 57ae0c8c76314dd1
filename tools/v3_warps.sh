#!/bin/bash
# K1 v3 compute-warp count sweep: each argument is one SZX_NVCC_FLAGS string; parity of the
# variant suite, then timings vs v1
for f in "$@"; do
  export SZX_NVCC_FLAGS="$f"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== flags: $f"
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "TestCompressVariants and 3" 2>&1 | tail -1
  K1_VARIANTS=1,3 python tools/k1_ab.py nyx1e-3 nyx1e-4 hacc noise hurricane
done
