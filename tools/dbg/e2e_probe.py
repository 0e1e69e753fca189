"""End-to-end (pinned host -> device -> host) pipelining variants at cfg2:
raw duplex copies, the library's run_bypass_host_bf16_pipelined, and a
three-stream schedule (H2D stream, compute stream, D2H stream, events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2411_00915_b200 as atmm
from paper_2411_00915_b200 import workloads

w = workloads.bypass_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
L = 4
reg = atmm.AdapterRegistry(L, w.d_in, w.d_out)
rng = np.random.default_rng(1)
for a, r in w.ranks.items():
    s = 1 / np.sqrt(r)
    reg.put(a, rng.uniform(-s, s, (L, w.d_in, r)).astype(np.float32), rng.uniform(-s, s, (L, r, w.d_out)).astype(np.float32))
plan = atmm.BypassPlan(reg, w.assignment)
steps, nbuf = 128, 6
xh = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16).uniform_(-1, 1).pin_memory() for _ in range(nbuf)]
yh = [torch.zeros(w.tokens, w.d_out, dtype=torch.bfloat16).pin_memory() for _ in range(nbuf)]
xs = [t.view(torch.int16).numpy().view(np.uint16) for t in xh]
ys = [t.view(torch.int16).numpy().view(np.uint16) for t in yh]

def t_api():
    a = [xs[i % nbuf] for i in range(steps)]; b = [ys[i % nbuf] for i in range(steps)]; l = [i % L for i in range(steps)]
    atmm.run_bypass_host_bf16_pipelined(plan, a[:3], b[:3], l[:3]); torch.cuda.synchronize()
    t = time.perf_counter(); atmm.run_bypass_host_bf16_pipelined(plan, a, b, l); torch.cuda.synchronize()
    return (time.perf_counter() - t) / steps * 1e6

K = int(os.environ.get("K", "4"))
dx = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device="cuda") for _ in range(K)]
dy = [torch.empty(w.tokens, w.d_out, dtype=torch.bfloat16, device="cuda") for _ in range(K)]
s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

def t_three(chunks=1):
    ev_in = [torch.cuda.Event() for _ in range(steps)]
    ev_c = [torch.cuda.Event() for _ in range(steps)]
    ev_out = [torch.cuda.Event() for _ in range(steps)]
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(steps):
        k = i % K
        with torch.cuda.stream(s_in):
            if i >= K: s_in.wait_event(ev_c[i - K])  # dx[k] free once the kernel of i-K ran
            dx[k].copy_(xh[i % nbuf], non_blocking=True)
            ev_in[i].record(s_in)
        with torch.cuda.stream(s_c):
            s_c.wait_event(ev_in[i])
            if i >= K: s_c.wait_event(ev_out[i - K])  # dy[k] free once its D2H ran
            dy[k].zero_()
            plan.apply(dx[k], dy[k], layer=i % L, stream=s_c)
            ev_c[i].record(s_c)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_c[i])
            yh[i % nbuf].copy_(dy[k], non_blocking=True)
            ev_out[i].record(s_out)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / steps * 1e6

def t_raw():
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(steps):
        with torch.cuda.stream(s_in): dx[i % K].copy_(xh[i % nbuf], non_blocking=True)
        with torch.cuda.stream(s_out): yh[i % nbuf].copy_(dy[i % K], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / steps * 1e6

for _ in range(2):
    t_api(); t_three(); t_raw()
print(w.name, "K", K, "api us/batch", round(min(t_api() for _ in range(3)), 1), "three-stream", round(min(t_three() for _ in range(3)), 1),
      "raw duplex copies", round(min(t_raw() for _ in range(3)), 1), flush=True)
