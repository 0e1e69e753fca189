#!/usr/bin/env python3
"""Eager launches of one ATMM kernel for ncu (no graph, no timing).

    python tools/profile_run.py --config cfg2 --iters 6
    python tools/profile_run.py --config cfg4 --iters 3
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--sm100", default=None, help="tile_m,cluster,bn,stages forced for every segment")
    args = ap.parse_args()
    import torch

    import paper_2411_00915_b200 as atmm
    from paper_2411_00915_b200.workloads import MergeWorkload, bypass_config

    rng = np.random.default_rng(0)
    if args.config == "cfg4":
        mw = MergeWorkload()
        L = args.layers
        reg = atmm.AdapterRegistry(L, mw.d_in, mw.d_out)
        s = 1.0 / np.sqrt(mw.rank)
        reg.put(1, rng.uniform(-s, s, (L, mw.d_in, mw.rank)).astype(np.float32),
                rng.uniform(-s, s, (L, mw.rank, mw.d_out)).astype(np.float32))
        W = torch.empty(L, mw.d_in, mw.d_out, dtype=torch.bfloat16, device="cuda").uniform_(-0.02, 0.02)
        for i in range(args.iters):
            atmm.merge_into(reg, 1, i % L, W[i % L], sign=1.0 if i % 2 == 0 else -1.0)
        torch.cuda.synchronize()
        return
    w = bypass_config(args.config)
    L = args.layers
    reg = atmm.AdapterRegistry(L, w.d_in, w.d_out)
    for a, r in w.ranks.items():
        s = 1.0 / np.sqrt(r)
        reg.put(a, rng.uniform(-s, s, (L, w.d_in, r)).astype(np.float32),
                rng.uniform(-s, s, (L, r, w.d_out)).astype(np.float32))
    table = None
    if args.sm100:
        lc = tuple(int(v) for v in args.sm100.split(","))
        table = atmm.TilingTable()
        for m in sorted(set(w.lengths.values())):
            for r in set(w.ranks.values()):
                table.insert(atmm.m_bucket_of(m), w.d_in, r, (128, 128, 256, 128, 16, 64), 1, sm100=lc)
    plan = atmm.BypassPlan(reg, w.assignment, table)
    xs = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1) for _ in range(L)]
    ys = [torch.zeros(w.tokens, w.d_out, dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    for i in range(args.iters):
        plan.apply(xs[i % L], ys[i % L], layer=i % L)
    torch.cuda.synchronize()
    print("launches/step, tiles, ctas:", plan.stats())


if __name__ == "__main__":
    main()
