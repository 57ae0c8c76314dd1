#!/bin/bash
# K1 on small fields (Hurricane 25M values, CESM-sized 6.5M) under build options
for f in "$@"; do
  export SZX_NVCC_FLAGS="$f"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" || continue
  echo "== flags: $f"
  python tools/kernel_times.py 25000000 | grep -E "compress|decode"
  python tools/kernel_times.py 6480000 | grep -E "compress|decode"
done
