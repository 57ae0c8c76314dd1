mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_large.py -x -q -k "batch" > gpurun_out/batch_tests.log 2>&1; echo rc=$? >> gpurun_out/batch_tests.log
timeout 300 python tools/bench_batch.py --reps 3 > gpurun_out/bench_batch.json 2>&1
