set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
for c in cfg2 cfg1 cfg3 cfg5 cfg4; do timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 300 gpurun_out/bench_$c.json; echo; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
timeout 300 python bench.py --config cfg4 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref4.json 2> gpurun_out/bench_ref4.err; tail -c 300 gpurun_out/bench_ref4.json
ATMM_BENCH_DIST=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-forward --no-cpu-baseline > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; tail -c 400 gpurun_out/bench_gloo2.json
bash tools/ncu_round.sh > gpurun_out/ncu_round.log 2>&1; ls gpurun_out/*.ncu-rep
