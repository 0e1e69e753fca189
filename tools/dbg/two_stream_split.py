"""Stress: split-path applies of one plan on several streams at once (each
stream its own scratch), many iterations -- does any grid wait on CTAs that
cannot become resident?  Prints the elapsed time; run under `timeout`."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2411_00915_b200 as atmm
from paper_2411_00915_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
nstreams = int(sys.argv[2]) if len(sys.argv) > 2 else 2
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 300
w = workloads.bypass_config(name)
reg = atmm.AdapterRegistry(1, w.d_in, w.d_out)
rng = np.random.default_rng(1)
for a, r in w.ranks.items():
    s = 1 / np.sqrt(r)
    reg.put(a, rng.uniform(-s, s, (1, w.d_in, r)).astype(np.float32), rng.uniform(-s, s, (1, r, w.d_out)).astype(np.float32))
plan = atmm.BypassPlan(reg, w.assignment)
print({g["path_bf16"] for g in plan.describe()}, flush=True)
xs = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1) for _ in range(nstreams)]
ys = [torch.zeros(w.tokens, w.d_out, dtype=torch.bfloat16, device="cuda") for _ in range(nstreams)]
streams = [torch.cuda.Stream() for _ in range(nstreams)]
torch.cuda.synchronize()
t0 = time.time()
for it in range(iters):
    for k in range(nstreams):
        with torch.cuda.stream(streams[k]):
            plan.apply(xs[k], ys[k], stream=streams[k])
torch.cuda.synchronize()
print(f"{name} streams={nstreams} iters={iters} ok {time.time() - t0:.2f}s", flush=True)
