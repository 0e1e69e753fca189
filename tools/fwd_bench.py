#!/usr/bin/env python3
"""Layer-forward microbenchmark: our fused forward (base GEMM + bypass as K
extension + tanh, forward_kernels.cu) against the unfused composition a
caller would otherwise run: cuBLAS x @ W (torch.mm, bf16) + our bypass
kernel into the fp32-free bf16 output + tanh; and against cuBLAS alone.

    python tools/fwd_bench.py [--configs cfg2,cfg3,cfg5] [--layers 4] [--reps 20]

Per-layer us, TFLOP/s (2 n d^2 + bypass FLOPs) and fraction of the measured
dense bf16 peak (MEASURED_PEAKS.json).  CUDA events, CUDA graphs, warm-up.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00915_b200 as atmm  # noqa: E402
from paper_2411_00915_b200.workloads import bypass_config  # noqa: E402


def timed(fn, reps, warm=3):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    with torch.cuda.stream(s):
        g.replay()
        torch.cuda.synchronize()
        for _ in range(5):
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg2,cfg3,cfg5")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = peaks["bf16_tflops"]
    for name in args.configs.split(","):
        w = bypass_config(name)
        L, d, n = args.layers, w.d_in, w.tokens
        rng = np.random.default_rng(0)
        reg = atmm.AdapterRegistry(L, d)
        for a, r in w.ranks.items():
            s = 1 / np.sqrt(r)
            reg.put(a, rng.uniform(-s, s, (L, d, r)).astype(np.float32), rng.uniform(-s, s, (L, r, d)).astype(np.float32))
        W = (torch.rand(L, d, d, device="cuda") * 2 - 1).mul_(1 / np.sqrt(d)).bfloat16()
        x = (torch.rand(n, d, device="cuda") * 2 - 1).bfloat16()
        plan = atmm.BypassPlan(reg, w.assignment)
        fw = atmm.LayerForward(plan)
        out = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
        flops = L * (2 * n * d * d + w.flops())
        t_ours = timed(lambda: fw.run(W, x, out), args.reps) / L
        merged = atmm.LayerForward(None, n=n, hidden_dim=d)
        t_merged = timed(lambda: merged.run(W, x, out), args.reps) / L
        bufs = [torch.empty(n, d, dtype=torch.bfloat16, device="cuda") for _ in range(2)]

        def unfused():
            cur = x
            for l in range(L):
                y = bufs[l % 2]
                torch.mm(cur, W[l], out=y)
                plan.apply(cur, y, layer=l)
                torch.tanh_(y)
                cur = y

        t_unf = timed(unfused, args.reps) / L

        def cublas():
            cur = x
            for l in range(L):
                torch.mm(cur, W[l], out=bufs[l % 2])
                cur = bufs[l % 2]

        t_cub = timed(cublas, args.reps) / L
        tf = lambda t: flops / L / (t * 1e-6) / 1e12  # noqa: E731
        print(json.dumps({"config": name, "n": n, "d": d, "layers": L, "stats": fw.stats(),
                          "us_per_layer": {"fused_forward": round(t_ours, 2), "merged_forward": round(t_merged, 2),
                                           "cublas_mm+bypass+tanh": round(t_unf, 2), "cublas_mm_only": round(t_cub, 2)},
                          "tflops_fused": round(tf(t_ours), 1), "frac_of_bf16_peak": round(tf(t_ours) / peak, 3),
                          "tflops_cublas_mm_only": round(2 * n * d * d / (t_cub * 1e-6) / 1e12, 1)}))


if __name__ == "__main__":
    main()
