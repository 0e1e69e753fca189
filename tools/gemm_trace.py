"""Per-CTA %globaltimer events of one atmm_gemm launch (replayed from a CUDA
graph after a warm-up launch of the same GEMM).

    python tools/gemm_trace.py 256x4096x4096 [--env ATMM_FWD_KZ=2 ...]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_00915_b200 as atmm  # noqa: E402
from paper_2411_00915_b200._lib import lib  # noqa: E402

EV = {0: "start", 7: "griddep released", 1: "first full", 2: "tile0 mma issued", 4: "tile0 tfull",
      5: "tile0 epi done", 6: "end"}


def main():
    m, k, n = (int(v) for v in sys.argv[1].split("x"))
    for kv in sys.argv[2:]:
        key, val = kv.split("=")
        os.environ[key] = val
    lib.atmm_debug_set_trace.argtypes = [ctypes.c_void_p]
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k**0.5
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(50):
        atmm.gemm(a, b, out=c)
    torch.cuda.synchronize()
    tr = torch.zeros(8192 * 16, dtype=torch.int64, device="cuda")
    lib.atmm_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(3):
                atmm.gemm(a, b, out=c)
    lib.atmm_debug_set_trace(None)
    for _ in range(3):
        tr.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
    t = tr.view(8192, 16).cpu().numpy()[4096:]
    live = t[:, 0] > 0
    t = t[live]
    t0 = t[:, 0].min()
    print(f"{m}x{k}x{n} CTAs traced: {live.sum()}")
    for e, name in EV.items():
        v = t[:, e]
        v = v[v > 0] - t0
        if v.size:
            print(f"  {name:18s} min {v.min() / 1e3:7.2f} us  median {np.median(v) / 1e3:7.2f}  max {v.max() / 1e3:7.2f}")


if __name__ == "__main__":
    main()
