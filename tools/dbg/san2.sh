CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
for tool in memcheck synccheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_run.py > gpurun_out/san/${tool}_r02.log 2>&1
  echo "== $tool rc=$?"; tail -3 gpurun_out/san/${tool}_r02.log
done
timeout 1200 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_run.py --only a2a > gpurun_out/san/racecheck_a2a_r02.log 2>&1; echo "== racecheck a2a rc=$?"; tail -3 gpurun_out/san/racecheck_a2a_r02.log
