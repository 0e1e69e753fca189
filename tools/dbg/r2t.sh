CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
timeout 900 $CS --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/san/memcheck_r02g.log 2>&1; echo "memcheck rc=$?"; tail -14 gpurun_out/san/memcheck_r02g.log
timeout 900 $CS --tool synccheck --print-limit 20 python tools/sanitize_run.py --small > gpurun_out/san/synccheck_r02g.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san/synccheck_r02g.log
timeout 900 $CS --tool racecheck --racecheck-report hazard --print-limit 10 python tools/sanitize_run.py --small --only a2a,overlap,chunks > gpurun_out/san/racecheck_a2a_r02g.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/san/racecheck_a2a_r02g.log
