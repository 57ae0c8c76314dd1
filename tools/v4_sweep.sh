#!/bin/bash
# K1 v4 build-parameter sweep: "boxes defer lb ahead" tuples, timed on NYX 1e-3, HACC and noise
for cfg in "$@"; do
  set -- $cfg
  export SZX_NVCC_FLAGS="-DSZX_V4_BOXES=$1 -DSZX_V4_DEFER=$2 -DSZX_V4_LB=$3 -DSZX_V4_AHEAD=$4"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== boxes $1 defer $2 lb $3 ahead $4"
  K1_VARIANTS=4 timeout 120 python tools/k1_ab.py nyx1e-3 hacc noise
done
