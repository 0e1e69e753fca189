"""Two independent split-path applies back to back (the second shrink starts
early); prints the split overlap counters.  For compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
import torch
import paper_2411_00915_b200 as atmm
from conftest import path_table

D = 1024
reg = atmm.AdapterRegistry(2, D, D)
rng = np.random.default_rng(1)
ranks = {0: 16, 1: 64, 2: 32}
for a, r in ranks.items():
    s = 1 / np.sqrt(r)
    reg.put(a, rng.uniform(-s, s, (2, D, r)).astype(np.float32), rng.uniform(-s, s, (2, r, D)).astype(np.float32))
asg = np.repeat(np.asarray(sorted(ranks), np.int32), 128)
asg = asg[np.random.default_rng(9).permutation(asg.size)]
plan = atmm.BypassPlan(reg, asg, path_table(atmm, asg, ranks, D, D, "split"))
print(plan.describe()[0]["split"], flush=True)
n = asg.size
bufs = [torch.empty(n, D, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1) for _ in range(4)]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    plan.apply(bufs[0], bufs[1], layer=0, stream=s)
    plan.apply(bufs[2], bufs[3], layer=1, stream=s)
s.synchronize()
print("ok", atmm.split_overlap_stats(), flush=True)
