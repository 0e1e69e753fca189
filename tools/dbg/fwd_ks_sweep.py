"""cfg1 / cfg2 fused layer forward over the shrink K split (ks) and GEMM
split-K (kz) options (atmm_gemm_opts), graph-timed like tools/fwd_bench.py."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tools"))
import numpy as np
import torch
import paper_2411_00915_b200 as atmm
from paper_2411_00915_b200.workloads import bypass_config
from fwd_bench import timed

for name in (sys.argv[1] if len(sys.argv) > 1 else "cfg1").split(","):
    w = bypass_config(name)
    n, d = w.tokens, w.d_in
    reg = atmm.AdapterRegistry(1, d, d)
    rng = np.random.default_rng(1)
    for a, r in w.ranks.items():
        s = 1 / np.sqrt(r)
        reg.put(a, rng.uniform(-s, s, (1, d, r)).astype(np.float32), rng.uniform(-s, s, (1, r, d)).astype(np.float32))
    plan = atmm.BypassPlan(reg, w.assignment)
    W = (torch.randn(1, d, d, device="cuda") / np.sqrt(d)).to(torch.bfloat16)
    x = torch.empty(n, d, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    out = torch.empty_like(x)
    for ks in (0, 1, 2, 4, 8, 16):
        for kz in (0, 2, 4, 8):
            try:
                fw = atmm.LayerForward(plan, opts={"ks": ks, "kz": kz})
                us = timed(lambda: fw.run(W, x, out), 20)
                st = fw.stats()
                print(name, "ks", ks, "kz", kz, "->", round(us, 2), "us", "(shrink_ks", st["shrink_ks"], "split_k", st["gemm_split_k"], ")", flush=True)
            except Exception as e:
                print(name, "ks", ks, "kz", kz, "ERR", str(e)[:80], flush=True)
