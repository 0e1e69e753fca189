timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_bypass.py tests/test_gpu_configs.py tests/test_gpu_sharding.py -q -x 2>&1 | tail -3
timeout 300 python tools/path_bench.py --configs cfg3,cfg5,cfg2 --paths auto 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['path'], d['us_per_step'], d['frac'])"
timeout 120 python tools/split_trace.py --config cfg3 --reps 1 2>&1 | tail -14
