timeout 200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_configs.py tests/test_gpu_bypass.py tests/test_gpu_sharding.py tests/test_gpu_rank_chunks.py -q -x 2>&1 | tail -2
timeout 120 python tools/split_trace.py --config cfg3 --reps 1 2>&1 | grep -v "ld issued" | tail -26
timeout 120 python tools/path_bench.py --configs cfg3,cfg5 --paths auto --steps 100 > gpurun_out/pb35.log 2>&1; cut -c1-160 gpurun_out/pb35.log
