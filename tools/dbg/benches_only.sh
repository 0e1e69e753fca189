for c in cfg2 cfg1 cfg3 cfg5 cfg4; do timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/r01i_bench_$c.json 2> gpurun_out/r01i_bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01i_bench_ref.json 2> gpurun_out/r01i_bench_ref.err
ls gpurun_out | grep r01i
