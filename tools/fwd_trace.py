#!/usr/bin/env python3
"""Per-CTA timeline of one layer-forward step (shrink + GEMM), %globaltimer.

    python tools/fwd_trace.py --config cfg2
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SH = {0: "shrink start", 1: "shrink griddep released", 2: "shrink loads issued", 3: "shrink mma first full",
      4: "shrink mma done", 5: "shrink epi done-wait ret", 6: "shrink epi done", 7: "shrink cluster sync1",
      8: "shrink reduce done", 9: "shrink end"}
GE = {0: "gemm start", 1: "gemm first full", 3: "gemm ext griddep released", 2: "gemm tile0 mma done",
      4: "gemm tile0 tfull", 5: "gemm tile0 epi done", 6: "gemm end"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--graph", action="store_true", help="replay the traced step from a CUDA graph")
    args = ap.parse_args()
    import torch

    import paper_2411_00915_b200 as atmm
    from paper_2411_00915_b200._lib import lib
    from paper_2411_00915_b200.workloads import bypass_config

    lib.atmm_debug_set_trace.argtypes = [ctypes.c_void_p]
    w = bypass_config(args.config)
    L, d = args.layers, w.d_in
    rng = np.random.default_rng(0)
    reg = atmm.AdapterRegistry(L, d)
    for a, r in w.ranks.items():
        s = 1.0 / np.sqrt(r)
        reg.put(a, rng.uniform(-s, s, (L, d, r)).astype(np.float32), rng.uniform(-s, s, (L, r, d)).astype(np.float32))
    W = (torch.rand(L, d, d, device="cuda") * 2 - 1).mul_(1 / np.sqrt(d)).bfloat16()
    x = (torch.rand(w.tokens, d, device="cuda") * 2 - 1).bfloat16()
    fw = atmm.LayerForward(atmm.BypassPlan(reg, w.assignment))
    print(fw.stats())
    out = fw.run(W, x)
    for _ in range(200):  # warm the clocks
        fw.run(W, x, out)
    torch.cuda.synchronize()
    tr = torch.zeros(8192 * 16, dtype=torch.int64, device="cuda")
    for rep in range(2):
        tr.zero_()
        torch.cuda.synchronize()
        lib.atmm_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
        if args.graph:  # launches from a CUDA graph: no host gaps between them
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                fw.run(W, x, out, num_layers=1)
            lib.atmm_debug_set_trace(None)
            tr.zero_()
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                g.replay()
        else:
            fw.run(W, x, out, num_layers=1)
        torch.cuda.synchronize()
        lib.atmm_debug_set_trace(None)
        raw = tr.cpu().numpy().reshape(8192, 16).astype(np.float64)
        ev = raw[:, :14]
        nz = ev[ev > 0]
        t0 = nz.min()
        print(f"rep {rep}:")
        g = raw[4096:4096 + 4096]
        ok = (g[:, 14] > 0) & (g[:, 15] > 0)
        if ok.any():
            mhz = (g[ok, 15] - g[ok, 14]) / (g[ok, 6] - g[ok, 0]) * 1e3
            print(f"  gemm SM clock during the kernel: median {np.median(mhz):.0f} MHz (min {mhz.min():.0f})")
        for base, evs in ((0, SH), (4096, GE)):
            for ev, name in evs.items():
                col = raw[base:base + 4096, ev]
                col = col[col > 0]
                if col.size == 0:
                    continue
                rel = (col - t0) / 1e3
                print(f"  {name:<28} n={col.size:4d} min {rel.min():7.2f} p10 {np.percentile(rel, 10):7.2f} "
                      f"med {np.median(rel):7.2f} p90 {np.percentile(rel, 90):7.2f} max {rel.max():7.2f} us")


if __name__ == "__main__":
    main()
