timeout 300 python -m pytest tests/test_gpu_bypass.py tests/test_gpu_shim.py tests/test_gpu_precise.py tests/test_gpu_shapes.py tests/test_gpu_fixture.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 50 --warmup 5 --no-forward --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['us_per_batch'], d['e2e_run_bypass'])"
