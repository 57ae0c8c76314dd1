timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_large.py -q -x -m gpu -k "batch or cesm or Batch" > gpurun_out/batchidx_pytest.log 2>&1
timeout 600 python bench.py --config cesm --steps 20 > gpurun_out/batchidx_cesm.json 2> gpurun_out/batchidx_cesm.err
