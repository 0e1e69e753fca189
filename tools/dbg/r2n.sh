timeout 300 python -m pytest tests/test_gpu_paths.py tests/test_gpu_configs.py tests/test_gpu_bypass.py tests/test_gpu_rank_chunks.py tests/test_gpu_sharding.py -q -x > gpurun_out/pytest_split.log 2>&1; tail -3 gpurun_out/pytest_split.log
timeout 120 python tools/path_bench.py --configs cfg3,cfg5 --paths auto --steps 100 > gpurun_out/pb35.log 2>&1; cut -c1-200 gpurun_out/pb35.log
timeout 60 python tools/split_trace.py --config cfg3 --reps 1 > gpurun_out/split_trace3.txt 2>&1; tail -28 gpurun_out/split_trace3.txt
