for o in '{"pair": 1, "kz": 1}' '{"pair": 0, "kz": 1}' '{"pair": 0, "bn": 256}' '{"pair": 1, "bn": 128}' '{"pair": 0, "stages": 2}' '{"pair": 0, "kz": 2}'; do
  for s in 300x1000x264 257x192x512 384x576x264 512x4096x4096; do
    CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/dbg/gemm_opts_probe.py $s "$o" 2>&1 | grep -E "max err|Error|error" | head -2
  done
done
