# cfg1 / cfg2 layer forward under the shrink K split and GEMM split-K knobs
for c in cfg1 cfg2; do
  for ks in 2 4 8 16; do
    for kz in 1 2 4 8; do
      r=$(ATMM_FWD_KS=$ks ATMM_FWD_KZ=$kz timeout 200 python tools/fwd_bench.py --configs $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_layer']['fused_forward'], d['stats']['shrink_ks'], d['stats']['gemm_split_k'])")
      echo "$c ks=$ks kz=$kz -> $r"
    done
  done
done
