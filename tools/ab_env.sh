#!/bin/bash
# A/B the bench across environment settings, interleaved, same box:
#   tools/ab_env.sh cfg2 3 "" "ATMM_NO_PDL=1" ...
cfg=$1; reps=$2; shift 2
for r in $(seq 1 $reps); do
  for e in "$@"; do
    v=$(env $e timeout 200 python bench.py --config $cfg --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-forward --group 1 --soak-s 0.3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_batch'] if 'us_per_batch' in d else d['ms_per_step']*1e3,3))")
    echo "$cfg rep$r [$e] us/step $v"
  done
done
