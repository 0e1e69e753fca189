"""One atmm_gemm (and one torch.matmul) call on a given shape, for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_00915_b200 as atmm  # noqa: E402

m, k, n = (int(v) for v in sys.argv[1].split("x"))
a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k**0.5
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    atmm.gemm(a, b, out=c)
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
