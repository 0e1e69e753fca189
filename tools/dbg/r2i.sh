timeout 600 python tools/step_timeline.py --config cfg2 --steps 10 --out gpurun_out/timeline_cfg2.json > gpurun_out/timeline_cfg2.txt 2>&1; tail -3 gpurun_out/timeline_cfg2.txt
timeout 900 python tools/path_bench.py --configs cfg1,cfg2 --paths auto > gpurun_out/path_bench.log 2>&1; cat gpurun_out/path_bench.log | cut -c1-160
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
