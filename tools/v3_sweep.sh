#!/bin/bash
# K1 v3 build-parameter sweep: "slots defer" pairs, timed on NYX 1e-3, HACC and noise
for cfg in "$@"; do
  set -- $cfg
  export SZX_NVCC_FLAGS="-DSZX_V3_SLOTS=$1 -DSZX_V3_DEFER=$2"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== slots $1 defer $2"
  K1_VARIANTS=3 python tools/k1_ab.py nyx1e-3 hacc noise
done
