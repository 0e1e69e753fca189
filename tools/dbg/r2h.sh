OUT=gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 400 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:atmm -c 200 --csv --log-file $OUT/launches_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --soak-s 0 --no-forward \
   > $OUT/launches_bench.log 2>&1
timeout 400 $NCU --set full --clock-control none --import-source on -k regex:atmm_bypass -s 4 -c 1 \
   -o $OUT/prof_cfg2 -f python tools/profile_run.py --config cfg2 --iters 6 > $OUT/ncu_cfg2.log 2>&1
for cfg in cfg3 cfg5; do
  timeout 400 $NCU --set full --clock-control none --import-source on -k regex:"atmm_(shrink|expand)" -s 4 -c 2 \
     -o $OUT/prof_$cfg -f python tools/profile_run.py --config $cfg --iters 6 > $OUT/ncu_$cfg.log 2>&1
done
ls -la $OUT
