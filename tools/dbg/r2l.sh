timeout 90 python tools/path_bench.py --configs cfg2 --paths auto --x-lsu 1 --steps 50 > gpurun_out/pb1.log 2>&1; cut -c1-150 gpurun_out/pb1.log; tail -2 gpurun_out/pb1.log | cut -c1-300
timeout 240 python tools/dbg/with_x_lsu.py tests/test_gpu_paths.py tests/test_gpu_bypass.py tests/test_gpu_configs.py tests/test_gpu_overlap.py tests/test_gpu_shapes.py tests/test_gpu_rank_chunks.py -q -x -m gpu > gpurun_out/pytest_xlsu.log 2>&1; tail -3 gpurun_out/pytest_xlsu.log
timeout 90 python tools/path_bench.py --configs cfg1,cfg2 --paths auto --x-lsu 1 > gpurun_out/pb1.log 2>&1; cut -c1-150 gpurun_out/pb1.log
timeout 90 python tools/path_bench.py --configs cfg2 --paths auto --x-lsu 1 --chain > gpurun_out/pb1c.log 2>&1; cut -c1-150 gpurun_out/pb1c.log
