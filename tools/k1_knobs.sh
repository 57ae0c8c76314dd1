#!/bin/bash
# K1 (v1 + v3) timing under build-flag variants: each argument is one SZX_NVCC_FLAGS string
for f in "$@"; do
  export SZX_NVCC_FLAGS="$f"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== flags: $f"
  K1_VARIANTS=1,3 python tools/k1_ab.py nyx1e-3 hacc noise
done
