timeout 900 python -m pytest tests/test_gpu_rank_chunks.py tests/test_gpu_mixture.py -q -x > gpurun_out/pytest_chunks.log 2>&1; tail -25 gpurun_out/pytest_chunks.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
