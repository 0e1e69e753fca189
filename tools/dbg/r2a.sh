set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02e.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02e.log
for c in cfg2 cfg3 cfg5 cfg1; do timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_r02e_$c.json 2> gpurun_out/bench_r02e_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r02e_ref.json 2> gpurun_out/bench_r02e_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02e.log 2>&1
