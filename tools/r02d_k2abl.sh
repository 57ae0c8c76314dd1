# K2 timing ablation: conflict-free column loads (wrong output) vs default
timeout 300 python tools/kernel_times.py > gpurun_out/k2abl_def.txt 2>&1
export SZX_NVCC_FLAGS="-DSZX_K2_ABL=1"
python -c "from paper_2201_13020_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
timeout 300 python tools/kernel_times.py > gpurun_out/k2abl_on.txt 2>&1
