set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "host or Fast or trunc or trailing or Errors or Golden" > gpurun_out/host_pytest.log 2>&1
timeout 300 python tools/e2e_pipeline.py 8 16 32 > gpurun_out/e2e_pipe.txt 2>&1
