timeout 300 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_paths.py tests/test_gpu_bypass.py tests/test_gpu_configs.py -q -x > gpurun_out/pytest_y.log 2>&1; tail -3 gpurun_out/pytest_y.log
timeout 120 python tools/path_bench.py --configs cfg1,cfg2 --paths auto > gpurun_out/pb2.log 2>&1; cut -c1-200 gpurun_out/pb2.log
timeout 120 python tools/path_bench.py --configs cfg2 --paths auto --chain > gpurun_out/pb2c.log 2>&1; cut -c1-200 gpurun_out/pb2c.log
timeout 120 python tools/step_timeline.py --config cfg2 --steps 10 --out gpurun_out/timeline_cfg2.json > gpurun_out/timeline_cfg2.txt 2>&1; tail -3 gpurun_out/timeline_cfg2.txt
