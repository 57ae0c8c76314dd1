# K1 input boxes with an L2 evict-first policy vs default
# ab_lib/libszx_evict.so = the library built here with SZX_NVCC_FLAGS="-DSZX_K1_EVICT=1" (untracked)
for i in 1 2; do
timeout 300 python tools/kernel_times.py > gpurun_out/evict_def$i.txt 2>&1
SZX_LIB=ab_lib/libszx_evict.so timeout 300 python tools/kernel_times.py > gpurun_out/evict_on$i.txt 2>&1
SZX_LIB=ab_lib/libszx_evict.so timeout 300 python tools/kernel_times.py 25000000 > gpurun_out/evict_on_hur$i.txt 2>&1
timeout 300 python tools/kernel_times.py 25000000 > gpurun_out/evict_def_hur$i.txt 2>&1
done
