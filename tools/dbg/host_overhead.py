"""Host-side cost of one eager apply (enqueue only, GPU not waited on)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_00915_b200 as atmm
from paper_2411_00915_b200.workloads import bypass_config
w = bypass_config("cfg2")
reg = atmm.AdapterRegistry(1, w.d_in, w.d_out)
rng = np.random.default_rng(0)
for a, r in w.ranks.items():
    reg.put(a, rng.uniform(-.1, .1, (1, w.d_in, r)).astype(np.float32), rng.uniform(-.1, .1, (1, r, w.d_out)).astype(np.float32))
plan = atmm.BypassPlan(reg, w.assignment)
x = torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
ys = [torch.empty(w.tokens, w.d_out, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
s = torch.cuda.Stream()
for _ in range(50):
    plan.apply(x, ys[0], stream=s)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for i in range(N):
    plan.apply(x, ys[i % 4], stream=s)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"python apply enqueue: {(t1 - t0) / N * 1e6:.2f} us/call; wall incl. GPU {(t2 - t0) / N * 1e6:.2f} us/call")
