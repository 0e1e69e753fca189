# Raw PCIe: H2D alone, D2H alone, both at once (separate streams), pinned 4 MiB chunks.
import torch, time
n = 64
h_in = [torch.empty(2 << 20, dtype=torch.int16).pin_memory() for _ in range(4)]
h_out = [torch.empty(2 << 20, dtype=torch.int16).pin_memory() for _ in range(4)]
d = [torch.empty(2 << 20, dtype=torch.int16, device='cuda') for _ in range(8)]
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h):
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(n):
        if h2d:
            with torch.cuda.stream(sa): d[i % 4].copy_(h_in[i % 4], non_blocking=True)
        if d2h:
            with torch.cuda.stream(sb): h_out[i % 4].copy_(d[4 + i % 4], non_blocking=True)
    torch.cuda.synchronize(); return time.perf_counter() - t
for _ in range(2): run(True, True)
for name, a, b in [("H2D", 1, 0), ("D2H", 0, 1), ("both", 1, 1)]:
    t = run(a, b)
    moved = n * 4 * (1 << 20) * (a + b)
    print(f"{name}: {t*1e6/n:.1f} us per 4 MiB step, {moved/t/1e9:.1f} GB/s total")
