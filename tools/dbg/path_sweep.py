# Which kernel path the launcher picks over a grid of shapes (bf16 / fp32 Y).
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2411_00915_b200 as atmm
from paper_2411_00915_b200._lib import lib
for d in (1024, 4096, 8192, 12288):
    for r in (8, 16, 64, 128):
        reg = atmm.AdapterRegistry(1, d, d)
        z1, z2 = np.zeros((d, r), np.float32), np.zeros((r, d), np.float32)
        for a in range(4):
            reg.put(a, z1, z2)
        for rows in (16, 32, 96, 128, 600):
            asg = np.repeat(np.arange(4, dtype=np.int32), rows)
            g = atmm.BypassPlan(reg, asg).describe()
            paths = sorted({x['path_bf16'] for x in g})
            sp = [x['split'] for x in g]
            print(f"d={d:5d} r={r:3d} rows/seg={rows:4d}: bf16 {paths} split={sp[0]}")
