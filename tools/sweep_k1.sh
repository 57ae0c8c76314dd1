#!/bin/bash
# Rebuild the library with each K1 ring configuration and time the kernels (GPU).
#   bash tools/sweep_k1.sh "-DSZX_K1_DEFER=4" "-DSZX_K1_DEFER=6 -DSZX_K1_IN=3" ...
for cfg in "$@"; do
  echo "== $cfg"
  SZX_NVCC_FLAGS="$cfg" python -m paper_2201_13020_b200._build > /dev/null || { echo build failed; continue; }
  python tools/kernel_times.py | head -1
  SZX_NVCC_FLAGS="$cfg -DSZX_STATS" python -m paper_2201_13020_b200._build > /dev/null
  python tools/compress_stats.py | tail -8
done
python -m paper_2201_13020_b200._build > /dev/null
