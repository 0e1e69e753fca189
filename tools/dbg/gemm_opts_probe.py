"""Runs atmm.gemm for one (m, k, n, opts) in-process; used to isolate a crash."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_00915_b200 as atmm  # noqa: E402

m, k, n = (int(v) for v in sys.argv[1].split("x"))
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else None
rng = np.random.default_rng(1)
a = torch.from_numpy(rng.uniform(-1, 1, (m, k)).astype(np.float32)).cuda().to(torch.bfloat16)
b = torch.from_numpy(rng.uniform(-1, 1, (k, n)).astype(np.float32)).cuda().to(torch.bfloat16)
for dt in (torch.bfloat16, torch.float32):
    c = atmm.gemm(a, b, out_dtype=dt, opts=opts)
    torch.cuda.synchronize()
    err = (c.float() - a.float() @ b.float()).abs().max().item()
    print(sys.argv[1], opts, dt, "max err", err, flush=True)
