#!/bin/bash
# Rebuild with each flag set and time the kernels (GPU): bash tools/sweep_k2.sh "-DX=1" ...
for cfg in "$@"; do
  echo "== $cfg"
  SZX_NVCC_FLAGS="$cfg" python -m paper_2201_13020_b200._build > /dev/null || { echo build failed; continue; }
  python tools/kernel_times.py | sed -n 2,3p
done
python -m paper_2201_13020_b200._build > /dev/null
