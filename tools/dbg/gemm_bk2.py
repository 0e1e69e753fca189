"""A/B of the 128-deep K stage GEMM (ATMM_GEMM_BK2, read once per process):
parity vs an fp64 product of the same bf16 inputs, then graph-timed speed."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2411_00915_b200 as atmm  # noqa: E402
from tools.gemm_sweep import graph_time  # noqa: E402

os.environ.update(ATMM_FWD_PAIR="0", ATMM_FWD_KZ="1")
for m, k, n in [(7, 64, 512), (130, 1024, 1024), (300, 192, 264), (512, 4096, 4096)]:
    rng = np.random.default_rng(m + k)
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    b = (rng.uniform(-1, 1, (k, n)) / np.sqrt(k)).astype(np.float32)
    at = torch.from_numpy(a).cuda().bfloat16()
    bt = torch.from_numpy(b).cuda().bfloat16()
    want = at.double().cpu().numpy() @ bt.double().cpu().numpy()
    got = atmm.gemm(at, bt, out_dtype=torch.float32).cpu().numpy()
    err = np.max(np.abs(got - want))
    print(f"parity {m}x{k}x{n}: max err {err:.3e} tol {1e-2 * max(1, np.max(np.abs(want))):.3e}",
          "OK" if err <= 1e-2 * max(1, np.max(np.abs(want))) else "FAIL")
for m in (128, 256, 512, 1024):
    for bn in ("128", "256"):
        os.environ["ATMM_FWD_BN"] = bn
        a = torch.randn(m, 4096, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16) / 64
        c = torch.empty(m, 4096, device="cuda", dtype=torch.bfloat16)
        print(f"time m={m} bn={bn}: {graph_time(lambda: atmm.gemm(a, b, out=c)) * 1e3:.2f} us")
