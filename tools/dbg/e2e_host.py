# Host enqueue cost vs wall time of the pipelined run_bypass (cfg2).
import sys, time, ctypes
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2411_00915_b200 as atmm
from paper_2411_00915_b200.workloads import bypass_config
w = bypass_config('cfg2')
reg = atmm.AdapterRegistry(4, w.d_in, w.d_out)
rng = np.random.default_rng(0)
for a, r in w.ranks.items():
    reg.put(a, rng.uniform(-.1, .1, (4, w.d_in, r)).astype(np.float32), rng.uniform(-.1, .1, (4, r, w.d_out)).astype(np.float32))
plan = atmm.BypassPlan(reg, w.assignment)
xs = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16).uniform_(-1, 1).pin_memory() for _ in range(6)]
ys = [torch.zeros(w.tokens, w.d_out, dtype=torch.bfloat16).pin_memory() for _ in range(6)]
xn = [t.view(torch.int16).numpy().view(np.uint16) for t in xs]
yn = [t.view(torch.int16).numpy().view(np.uint16) for t in ys]
N = 64
sx = [xn[i % 6] for i in range(N)]; sy = [yn[i % 6] for i in range(N)]; sl = [i % 4 for i in range(N)]
atmm.run_bypass_host_bf16_pipelined(plan, sx[:4], sy[:4], sl[:4])
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    atmm.run_bypass_host_bf16_pipelined(plan, sx, sy, sl)
    t1 = time.perf_counter()
    print(f"pipelined: {(t1 - t0) / N * 1e6:.1f} us per batch (wall, includes the final sync)")
# host cost of one apply (device buffers): enqueue only
xd = xs[0].cuda(); yd = ys[0].cuda()
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(N): plan.apply(xd, yd, layer=i % 4)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"apply enqueue: {(t1 - t0) / N * 1e6:.1f} us per call, gpu drain {(t2 - t1)*1e6:.0f} us")
