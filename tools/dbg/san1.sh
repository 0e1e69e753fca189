CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
timeout 300 python tools/sanitize_run.py > gpurun_out/san/plain.log 2>&1; tail -12 gpurun_out/san/plain.log
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 50 python tools/sanitize_run.py > gpurun_out/san/$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/san/$tool.log
done
