# K2 with 3 CTAs per SM (2 stages, 40 registers) vs the default 2 CTAs x 3 stages
# ab_lib/libszx_k2c3.so = the library built here with SZX_NVCC_FLAGS="-DSZX_K2_CTAS=3 -DSZX_K2_STAGES=2" (untracked)
set -x
for i in 1 2; do
timeout 300 python tools/kernel_times.py > gpurun_out/k2c3_new$i.txt 2>&1
SZX_LIB=ab_lib/libszx_k2c3.so timeout 300 python tools/kernel_times.py > gpurun_out/k2c3_c3_$i.txt 2>&1
done
