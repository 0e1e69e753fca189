CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
timeout 900 $CS --tool memcheck --print-limit 30 python tools/sanitize_run.py > gpurun_out/san/memcheck_r02.log 2>&1
echo "== memcheck rc=$?"; tail -3 gpurun_out/san/memcheck_r02.log; grep "Device Frame" gpurun_out/san/memcheck_r02.log | sort | uniq -c
timeout 600 python -m pytest tests/test_gpu_forward.py -q -x 2>&1 | tail -2
