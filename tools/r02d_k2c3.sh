# K2 with 3 CTAs per SM (2 stages, 40 registers) vs the default 2 CTAs x 3 stages
set -x
for i in 1 2; do
timeout 300 python tools/kernel_times.py > gpurun_out/k2c3_new$i.txt 2>&1
SZX_LIB=ab_lib/libszx_k2c3.so timeout 300 python tools/kernel_times.py > gpurun_out/k2c3_c3_$i.txt 2>&1
done
