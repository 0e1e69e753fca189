import numpy as np, torch, os, sys
sys.path.insert(0, '.')
import paper_2411_00915_b200 as atmm
d = 8192
reg = atmm.AdapterRegistry(1, d, d)
rng = np.random.default_rng(0)
for a in range(32):
    reg.put(a, rng.uniform(-.1, .1, (d, 128)).astype(np.float32), rng.uniform(-.1, .1, (128, d)).astype(np.float32))
asg = np.repeat(np.arange(32, dtype=np.int32), 128)[rng.permutation(4096)]
x = torch.empty(4096, d, dtype=torch.bfloat16, device='cuda').uniform_(-1, 1)
y = torch.zeros(4096, d, dtype=torch.bfloat16, device='cuda')
for path in ['split', 'fused']:
    os.environ['ATMM_PATH'] = path
    plan = atmm.BypassPlan(reg, asg)
    for _ in range(3): plan.apply(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [plan.apply(x, y) for _ in range(20)]; e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    byt = 4096 * d * 2 * 3 + 32 * 2 * d * 128 * 2
    print(path, plan.describe()[0]['path_bf16'], round(us, 1), 'us', round(byt / us / 1e3, 0), 'GB/s')
