timeout 600 python -m pytest tests/test_gpu_overlap.py -q -x > gpurun_out/pytest_overlap.log 2>&1; tail -15 gpurun_out/pytest_overlap.log
timeout 600 python tools/step_timeline.py --config cfg2 --steps 10 --out gpurun_out/timeline_cfg2.json > gpurun_out/timeline_cfg2.txt 2>&1; cat gpurun_out/timeline_cfg2.txt
timeout 600 python tools/path_bench.py --configs cfg1,cfg2 --paths auto > gpurun_out/path_bench.log 2>&1; tail -4 gpurun_out/path_bench.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
