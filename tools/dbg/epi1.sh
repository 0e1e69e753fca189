timeout 600 python -m pytest tests/test_gpu_paths.py tests/test_gpu_bypass.py tests/test_gpu_configs.py -q -x 2>&1 | tail -3
timeout 300 python tools/path_bench.py --configs cfg2,cfg1,cfg3,cfg5 --paths auto 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['path'], d['us_per_step'], d['frac'])"
