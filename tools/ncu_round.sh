#!/bin/bash
# Profiling pass for one round (run under gpurun).  Outputs in gpurun_out/.
set -x
OUT=gpurun_out
NCU=/usr/local/cuda/bin/ncu
for cfg in cfg2 cfg3 cfg5 cfg4; do
  timeout 300 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -c 12 --csv --log-file $OUT/launches_$cfg.csv python tools/profile_run.py --config $cfg --iters 6 > /dev/null 2>&1
done
timeout 400 $NCU --set full --clock-control none --import-source on -k regex:atmm_bypass -s 2 -c 1 \
   -o $OUT/prof_cfg2 -f python tools/profile_run.py --config cfg2 --iters 4 > $OUT/ncu_cfg2.log 2>&1
timeout 400 $NCU --set full --clock-control none --import-source on -k regex:atmm_bypass -s 2 -c 1 \
   -o $OUT/prof_cfg5 -f python tools/profile_run.py --config cfg5 --iters 4 > $OUT/ncu_cfg5.log 2>&1
timeout 400 $NCU --set full --clock-control none --import-source on -k regex:atmm_merge -s 2 -c 1 \
   -o $OUT/prof_cfg4 -f python tools/profile_run.py --config cfg4 --iters 4 > $OUT/ncu_cfg4.log 2>&1
ls -la $OUT
