timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for c in cfg2 cfg1 cfg3 cfg5 cfg4; do timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --config cfg4 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref4.json 2> gpurun_out/bench_ref4.err
timeout 120 python tools/step_timeline.py --config cfg2 --steps 10 --out gpurun_out/timeline_cfg2.json > gpurun_out/timeline_cfg2.txt 2>&1
python - <<'PY'
import json
for c in ["cfg2","cfg1","cfg3","cfg5","cfg4","ref","ref4"]:
    d=json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
    r=d.get("roofline") or {}
    print(c, d.get("impl"), round(d.get("value",0),3), d.get("ms_per_step"), r.get("frac"), (d.get("e2e") or {}).get("value"), (d.get("clocks") or {}).get("reasons"))
PY
