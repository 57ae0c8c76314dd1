#!/bin/bash
# K2 (decode) timing under build-flag variants: each argument is one SZX_NVCC_FLAGS string
for f in "$@"; do
  export SZX_NVCC_FLAGS="$f"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== flags: $f"
  python tools/kernel_times.py | grep -v "^compress"
  python tools/kernel_times.py 280953867 | grep decode
done
