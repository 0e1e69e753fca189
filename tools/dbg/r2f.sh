timeout 600 python tools/step_timeline.py --config cfg2 --steps 10 --out gpurun_out/timeline_cfg2.json > gpurun_out/timeline_cfg2.txt 2>&1; tail -4 gpurun_out/timeline_cfg2.txt
timeout 900 python tools/path_bench.py --configs cfg1,cfg2 --paths auto > gpurun_out/path_bench.log 2>&1; cat gpurun_out/path_bench.log | cut -c1-200
timeout 900 python tools/path_bench.py --configs cfg2 --paths auto --chain > gpurun_out/path_bench_chain.log 2>&1; cat gpurun_out/path_bench_chain.log | cut -c1-200
