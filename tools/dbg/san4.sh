CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
for fam in split stream fused merge forward gemm; do
  timeout 900 $CS --tool racecheck --racecheck-report hazard --print-limit 10 python tools/sanitize_run.py --small --only $fam > gpurun_out/san/racecheck_${fam}_r02.log 2>&1
  echo "== racecheck $fam rc=$?"; tail -2 gpurun_out/san/racecheck_${fam}_r02.log
done
