#!/bin/bash
# Profiling pass for one round (run under gpurun, 1 GPU).  Outputs in gpurun_out/.
#   launches_bench.csv : every kernel launch of a short bench.py run (cold, serialised)
#   prof_<cfg>.ncu-rep : one --set full capture of the dominant kernel per config
OUT=gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 400 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:atmm -c 200 --csv --log-file $OUT/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --soak-s 0 --no-forward \
   > $OUT/launches_bench.log 2>&1
# one step of each config: the a2a / fused kernel (1 launch) or the split pair
# (shrink + expand, 2 launches; ncu_summarize.py sums them)
timeout 400 $NCU --set full --clock-control none --import-source on -k regex:atmm_bypass -s 4 -c 1 \
   -o $OUT/prof_cfg2 -f python tools/profile_run.py --config cfg2 --iters 6 > $OUT/ncu_cfg2.log 2>&1
for cfg in cfg3 cfg5; do
  timeout 400 $NCU --set full --clock-control none --import-source on -k regex:"atmm_(shrink|expand)" -s 4 -c 2 \
     -o $OUT/prof_$cfg -f python tools/profile_run.py --config $cfg --iters 6 > $OUT/ncu_$cfg.log 2>&1
done
timeout 400 $NCU --set full --clock-control none --import-source on -k regex:atmm_merge -s 2 -c 1 \
   -o $OUT/prof_cfg4 -f python tools/profile_run.py --config cfg4 --iters 4 > $OUT/ncu_cfg4.log 2>&1
# layer forward (model.hpp:216-246): launch list + one full capture of each kernel at cfg2 / cfg5
timeout 300 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
   -k regex:fwd_ -c 60 --csv --log-file $OUT/launches_forward.csv python tools/fwd_bench.py --configs cfg2,cfg5 --layers 1 --reps 1 \
   > $OUT/launches_forward.log 2>&1
for cfg in cfg2 cfg5; do
  timeout 400 $NCU --set full --clock-control none --import-source on -k regex:"fwd_(shrink|gemm)" -s 2 -c 2 \
     -o $OUT/prof_fwd_$cfg -f python tools/fwd_bench.py --configs $cfg --layers 1 --reps 1 > $OUT/ncu_fwd_$cfg.log 2>&1
done
ls -la $OUT
