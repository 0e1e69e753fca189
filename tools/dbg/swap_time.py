# Adapter swap timing: raw pinned H2D vs put_async (cfg4 shapes: 32 layers, 4096 x 11008, r64).
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2411_00915_b200 as atmm
L, di, do, r = 32, 4096, 11008, 64
dn = torch.empty(L, di, r).uniform_(-.1, .1).pin_memory()
up = torch.empty(L, r, do).uniform_(-.1, .1).pin_memory()
buf = torch.empty(dn.numel() + up.numel(), device='cuda')
s = torch.cuda.Stream()
reg = atmm.AdapterRegistry(L, di, do)
for rep in range(4):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        e[0].record(s)
        buf[:dn.numel()].copy_(dn.view(-1), non_blocking=True)
        buf[dn.numel():].copy_(up.view(-1), non_blocking=True)
        e[1].record(s)
        reg.put_async(2, dn, up, stream=s)
        e[2].record(s)
    torch.cuda.synchronize()
    print(f"rep {rep}: raw H2D {e[0].elapsed_time(e[1]):.2f} ms ({(dn.numel()+up.numel())*4/e[0].elapsed_time(e[1])/1e6:.1f} GB/s), put_async {e[1].elapsed_time(e[2]):.2f} ms")
