set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
bash tools/ncu_round.sh > gpurun_out/ncu_round.log 2>&1
for c in cfg2 cfg1 cfg3 cfg5 cfg4 paper_in1 paper_in2; do timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
ls gpurun_out
