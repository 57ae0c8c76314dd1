# K1 / K2 time vs field size (smooth ridges, rel 1e-3): fixed cost and steady per-tile rate
for n in 33554432 67108864 134217728 268435456 536870912 1073741824 2147483648; do
  echo "n=$n"
  timeout 300 python tools/kernel_times.py $n | grep -E "compress|decode"
done
