#!/bin/bash
# Rebuild with each flag set and time all three kernels (GPU): bash tools/sweep_all.sh "-DX=1" ...
for cfg in "$@"; do
  echo "== $cfg"
  SZX_NVCC_FLAGS="$cfg" python -m paper_2201_13020_b200._build > /dev/null || { echo build failed; continue; }
  python tools/kernel_times.py | sed -n 1,3p
done
python -m paper_2201_13020_b200._build > /dev/null
