timeout 300 python -m pytest tests/test_gpu_bypass.py tests/test_gpu_shim.py tests/test_gpu_precise.py tests/test_gpu_paths.py -q -x > gpurun_out/pytest_host.log 2>&1; tail -3 gpurun_out/pytest_host.log
timeout 300 python bench.py --steps 100 --warmup 5 --no-forward --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'], d['e2e_run_bypass'], d['dependent_chain'], d['overlap'])"
