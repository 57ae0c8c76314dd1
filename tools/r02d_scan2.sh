# K1 with 2 look-back warps + 1 write-out warp (20 warps, 96 registers) vs default (1 + 2)
for F in "" "-DSZX_K1_SCAN=2 -DSZX_K1_WRITERS=1"; do
  export SZX_NVCC_FLAGS="$F"
  python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "== flags: $F"
  for n in 25000000 134217728 536870912; do
    timeout 300 python tools/kernel_times.py $n | grep -E "compress K1"
  done
  K1_VARIANTS=1,1 timeout 300 python tools/k1_ab.py hacc noise | cut -c1-160
done
