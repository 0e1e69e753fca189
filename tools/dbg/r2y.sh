timeout 300 python -m pytest tests/test_gpu_paths.py tests/test_gpu_configs.py tests/test_gpu_bypass.py -q -x 2>&1 | tail -2
timeout 120 python tools/path_bench.py --configs cfg3,cfg5 --paths auto --steps 100 > gpurun_out/pb35.log 2>&1; cut -c1-160 gpurun_out/pb35.log
