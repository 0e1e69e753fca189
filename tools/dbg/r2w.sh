timeout 300 python -m pytest tests/test_gpu_paths.py tests/test_gpu_configs.py tests/test_gpu_bypass.py tests/test_gpu_sharding.py tests/test_gpu_rank_chunks.py tests/test_gpu_mixture.py -q -x 2>&1 | tail -2
timeout 120 python tools/split_trace.py --config cfg5 --reps 1 2>&1 | grep -v "ld issued" | grep "expand\|shrink end" | head -12
timeout 120 python tools/path_bench.py --configs cfg3,cfg5 --paths auto --steps 100 > gpurun_out/pb35.log 2>&1; cut -c1-160 gpurun_out/pb35.log
