#!/bin/bash
# SASS of one kernel from the built library: tools/sass_fn.sh <mangled-name-substring>
cuobjdump -sass paper_2201_13020_b200/_lib/libszx_b200.so 2>/dev/null |
  awk -v pat="$1" '/Function :/ {on = index($0, pat) > 0} on'
