timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/path_bench.py --configs cfg1,cfg2,cfg3,cfg5 --paths auto,a2a,split,stream > gpurun_out/path_bench.log 2>&1; tail -30 gpurun_out/path_bench.log
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; cat gpurun_out/bench_cfg2.json
