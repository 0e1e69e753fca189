# A/B of 128-deep K stages on 2-SM pairs (ATMM_PAIR_BK2)
for v in 0 1; do
  echo "ATMM_PAIR_BK2=$v"
  ATMM_PAIR_BK2=$v timeout 300 python -c "
import sys,torch; sys.path.insert(0,'.')
import paper_2411_00915_b200 as atmm
from tools.gemm_sweep import graph_time
for m,k,n in ((1024,4096,4096),(2048,4096,4096),(4096,4096,4096),(8192,5120,5120)):
    a=torch.randn(m,k,device='cuda',dtype=torch.bfloat16); b=torch.randn(k,n,device='cuda',dtype=torch.bfloat16)/64
    c=torch.empty(m,n,device='cuda',dtype=torch.bfloat16)
    print(m,k,n, round(graph_time(lambda: atmm.gemm(a,b,out=c))*1e3,2), round(graph_time(lambda: torch.matmul(a,b,out=c))*1e3,2))
"
  ATMM_PAIR_BK2=$v timeout 300 python tools/fwd_bench.py --configs cfg3,cfg5 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['us_per_layer'], d['stats']['gemm_cta_group'])"
done
