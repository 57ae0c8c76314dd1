#!/bin/bash
# K1v2 build-parameter sweep: build each variant ("warps defer"), A/B against v1
for cfg in "$@"; do
  set -- $cfg
  export SZX_NVCC_FLAGS="-DSZX_K1V2_WARPS=$1 -DSZX_K1V2_DEFER=$2"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== warps $1 defer $2"
  python tools/k1_ab.py nyx1e-3 hacc noise
done
