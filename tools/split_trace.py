#!/usr/bin/env python3
"""Per-CTA timeline of the split path (shrink + expand), %globaltimer events.

    python tools/split_trace.py --config cfg3
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
EV = {0: "shrink start", 4: "shrink mma item0 full", 5: "shrink mma item1 full",
      **{16 + j: f"shrink ld issued item{j}" for j in range(12)},
      1: "shrink loaders done", 2: "shrink epilogue done", 3: "shrink end",
      8: "expand start", 13: "expand epi griddep returned", 14: "expand reduce done", 15: "expand grid barrier passed",
      12: "expand loaders see mid ready", 9: "expand loaders done", 10: "expand epilogue done",
      11: "expand end"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch

    import paper_2411_00915_b200 as atmm
    from paper_2411_00915_b200._lib import lib
    from paper_2411_00915_b200.workloads import bypass_config

    lib.atmm_debug_set_trace.argtypes = [ctypes.c_void_p]
    w = bypass_config(args.config)
    rng = np.random.default_rng(0)
    reg = atmm.AdapterRegistry(1, w.d_in, w.d_out)
    for a, r in w.ranks.items():
        s = 1.0 / np.sqrt(r)
        reg.put(a, rng.uniform(-s, s, (1, w.d_in, r)).astype(np.float32),
                rng.uniform(-s, s, (1, r, w.d_out)).astype(np.float32))
    plan = atmm.BypassPlan(reg, w.assignment)
    x = torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y = torch.zeros(w.tokens, w.d_out, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    tr = torch.zeros(1024 * 32, dtype=torch.int64, device="cuda")
    plan.apply(x, y)
    torch.cuda.synchronize()
    for rep in range(args.reps):
        flush.fill_(rep)
        tr.zero_()
        torch.cuda.synchronize()
        lib.atmm_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
        plan.apply(x, y)
        torch.cuda.synchronize()
        lib.atmm_debug_set_trace(None)
        raw = tr.cpu().numpy().reshape(1024, 32).astype(np.float64)
        t0 = raw[:, 0][raw[:, 0] > 0].min()
        print(f"rep {rep}:")
        for ev, name in EV.items():
            col = raw[:, ev]
            col = col[col > 0]
            if col.size == 0:
                continue
            rel = (col - t0) / 1e3
            print(f"  {name:<26} n={col.size:4d} min {rel.min():7.2f} p10 {np.percentile(rel, 10):7.2f} "
                  f"med {np.median(rel):7.2f} p90 {np.percentile(rel, 90):7.2f} max {rel.max():7.2f} us")
        # per-CTA expand: items, Y bytes vs the time its loaders finish
        sel = raw[:, 9] > 0
        if sel.any():
            items, yb = raw[sel, 20], raw[sel, 21]
            start, done = (raw[sel, 8] - t0) / 1e3, (raw[sel, 9] - t0) / 1e3
            order = np.argsort(done)
            print("  expand per CTA (slowest 8 / fastest 4): [cta, items, Y KB, start us, loaders done us]")
            idx = np.nonzero(sel)[0]
            for k in list(order[-8:]) + list(order[:4]):
                print(f"    {idx[k]:4d} {int(items[k]):3d} {yb[k] / 1024:7.1f} {start[k]:7.2f} {done[k]:7.2f}")
            print(f"  corr(Y bytes, done) = {np.corrcoef(yb, done)[0, 1]:.2f}  corr(start, done) = {np.corrcoef(start, done)[0, 1]:.2f}")


if __name__ == "__main__":
    main()
