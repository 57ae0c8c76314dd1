# f32x2 packed adds in K1 pass 1 and K2: parity subset + A/B kernel times
# ab_lib/libszx_nof2.so = the library built here with SZX_NVCC_FLAGS="-DSZX_K2_F2=0 -DSZX_K1_F2=0" (untracked)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "Golden or random_fields or FastBlock or K1Index or CompressVariants or mixed" > gpurun_out/f2_pytest.log 2>&1
for i in 1 2; do
timeout 300 python tools/kernel_times.py > gpurun_out/f2_kt_new$i.txt 2>&1
SZX_LIB=ab_lib/libszx_nof2.so timeout 300 python tools/kernel_times.py > gpurun_out/f2_kt_old$i.txt 2>&1
done
