#!/bin/bash
# A/B the bench across in-tree library builds (tools/ab/libatmm_b200_<tag>.so),
# interleaved, same box:  tools/ab_bench.sh cfg2 3 tagA tagB ...
cfg=$1; reps=$2; shift 2
for r in $(seq 1 $reps); do
  for tag in "$@"; do
    v=$(ATMM_LIB_VARIANT=$tag timeout 200 python bench.py --config $cfg --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --soak-s 0.3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_batch'] if 'us_per_batch' in d else d['ms_per_step']*1e3,3))")
    echo "$cfg rep$r $tag us/step $v"
  done
done
