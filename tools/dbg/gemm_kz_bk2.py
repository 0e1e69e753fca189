"""Graph-timed atmm_gemm at small m over the split-K setting (ATMM_FWD_KZ), 1-SM tiles."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_00915_b200 as atmm  # noqa: E402
from tools.gemm_sweep import graph_time  # noqa: E402

os.environ["ATMM_FWD_PAIR"] = "0"
for m in (64, 128, 256, 512):
    a = torch.randn(m, 4096, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16) / 64
    c = torch.empty(m, 4096, device="cuda", dtype=torch.bfloat16)
    want = torch.matmul(a, b).float()
    row = [m]
    for kz in ("1", "2", "4", "8"):
        os.environ["ATMM_FWD_KZ"] = kz
        t = graph_time(lambda: atmm.gemm(a, b, out=c))
        err = (c.float() - want).abs().max().item()
        row.append(f"kz{kz}={t * 1e3:.2f}us(err {err:.3f})")
    os.environ.pop("ATMM_FWD_KZ")
    row.append(f"auto={graph_time(lambda: atmm.gemm(a, b, out=c)) * 1e3:.2f}")
    print(*row)
