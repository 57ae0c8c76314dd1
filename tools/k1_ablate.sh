#!/bin/bash
# K1 v1 timing ablations (wrong output, timing only): each argument is an SZX_K1_ABL mask
for m in "$@"; do
  export SZX_NVCC_FLAGS="-DSZX_K1_ABL=$m"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== ablation mask $m"
  K1_VARIANTS=1 timeout 120 python tools/k1_ab.py nyx1e-3 hacc
done
