timeout 300 python -m pytest tests/test_gpu_paths.py -q -x -k "stream" 2>&1 | tail -3
timeout 300 python tools/path_bench.py --configs cfg2,cfg1,cfg3,cfg5 --paths auto,stream 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['path'], d['us_per_step'], d['frac'], d['max_abs_diff_vs_first'])"
timeout 120 python tools/stream_trace.py --config cfg2 | tail -13
