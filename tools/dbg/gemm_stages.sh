for st in 2 3 4 5 7 8; do
  for cfg in "0 128 1" "1 128 1" "0 256 1"; do set -- $cfg
    r=$(ATMM_GEMM_STAGES=$st ATMM_FWD_PAIR=$1 ATMM_FWD_BN=$2 ATMM_FWD_KZ=$3 timeout 200 python -c "
import torch,sys; sys.path.insert(0,'.')
import paper_2411_00915_b200 as atmm
from tools.gemm_sweep import graph_time
a=torch.randn(512,4096,device='cuda',dtype=torch.bfloat16); b=torch.randn(4096,4096,device='cuda',dtype=torch.bfloat16)
c=torch.empty(512,4096,device='cuda',dtype=torch.bfloat16)
print(round(graph_time(lambda: atmm.gemm(a,b,out=c))*1e3,2))" 2>&1 | tail -1)
    echo "stages=$st pair=$1 bn=$2 us=$r"
  done
done
