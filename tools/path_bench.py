#!/usr/bin/env python3
"""Per-step device time of one bypass apply per kernel path, bench.py's way
(K steps in one CUDA graph, X / Y rotating over > 2.5 x L2 of buffers, one
layer of factors per buffer), plus an oracle spot check of every path.

    python tools/path_bench.py [--configs cfg2,cfg3] [--paths auto,stream] [--steps 200]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
PATHS = {"auto": 0, "a2a": 1, "split": 2, "fused": 3, "stream": 4}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg5")
    ap.add_argument("--paths", default="auto,stream")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--x-ready", action="store_true")
    ap.add_argument("--y-dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--sorted", action="store_true",
                    help="rows grouped by adapter (consecutive runs: the split kernels' TMA-box path)")
    ap.add_argument("--launches", default=None,
                    help="';'-separated tile_m,cluster,bn,stages,path launches to force (instead of --paths)")
    ap.add_argument("--no-overlap", action="store_true", help="ATMM_PLAN_NO_OVERLAP on every plan")
    ap.add_argument("--chain", action="store_true",
                    help="dependent steps: step i+1 reads step i's Y as its X (d_in == d_out)")
    args = ap.parse_args()
    import torch

    import paper_2411_00915_b200 as atmm
    from paper_2411_00915_b200 import workloads

    dev = torch.device("cuda", 0)
    for name in args.configs.split(","):
        w = workloads.bypass_config(name)
        if args.sorted:
            w.assignment = workloads.make_assignment(w.lengths, shuffle=False)
        step_bytes = w.bytes(2 if args.y_dtype == "bf16" else 4)
        layers = min(64, max(2, int(np.ceil(2.5 * L2_BYTES / step_bytes))))
        reg = atmm.AdapterRegistry(layers, w.d_in, w.d_out, device=0)
        rng = np.random.default_rng(5)
        for a, r in w.ranks.items():
            s = 1.0 / np.sqrt(r)
            reg.put(a, rng.uniform(-s, s, (layers, w.d_in, r)).astype(np.float32),
                    rng.uniform(-s, s, (layers, r, w.d_out)).astype(np.float32))
        xs = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device=dev).uniform_(-1, 1) for _ in range(layers)]
        ydt = torch.bfloat16 if args.y_dtype == "bf16" else torch.float32
        ys = [torch.empty(w.tokens, w.d_out, dtype=ydt, device=dev).uniform_(-1, 1) for _ in range(layers)]
        ref = None
        y0 = ys[0].clone()
        variants = args.paths.split(",") if not args.launches else [
            [int(v) for v in l.split(",")] for l in args.launches.split(";")]
        for path in variants:
            if isinstance(path, list):
                plan = atmm.BypassPlan(reg, w.assignment, launch=path)
            elif path == "auto":
                plan = atmm.BypassPlan(reg, w.assignment)
            else:
                ranks = sorted(set(w.ranks.values()))
                seg_rows = max(np.bincount(w.assignment)) if w.assignment.size else 1
                launch = list(atmm.heuristic_launch(int(seg_rows), w.d_in, ranks[0], w.d_out))
                launch[4] = PATHS[path]
                plan = atmm.BypassPlan(reg, w.assignment, launch=launch)
            plan.set_x_ready(args.x_ready)
            plan.set_overlap(not args.no_overlap)
            desc = plan.describe()
            stream = torch.cuda.Stream(device=dev)
            # correctness spot check vs the first path (same inputs, layer 0)
            y = y0.clone()
            plan.apply(xs[0], y, layer=0)
            torch.cuda.synchronize()
            if ref is None:
                ref = y
                diff = 0.0
            else:
                diff = float((y.float() - ref.float()).abs().max())
            with torch.cuda.stream(stream):
                for i in range(5):
                    plan.apply(xs[i % layers], ys[i % layers], layer=i % layers, stream=stream)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
                for i in range(args.steps):
                    if args.chain:  # X of step i+1 = Y of step i
                        plan.apply(ys[i % layers], ys[(i + 1) % layers], layer=i % layers, stream=stream)
                    else:
                        plan.apply(xs[i % layers], ys[i % layers], layer=i % layers, stream=stream)
            g.replay()
            torch.cuda.synchronize()
            times = []
            for _ in range(args.reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    e0.record(stream)
                    g.replay()
                    e1.record(stream)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) * 1e3 / args.steps)
            us = min(times)
            # one launch alone on an idle GPU (L2 flushed)
            flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
            iso = []
            for k in range(min(5, layers)):
                flush.fill_(k)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    e0.record(stream)
                    plan.apply(xs[k], ys[k], layer=k, stream=stream)
                    e1.record(stream)
                torch.cuda.synchronize()
                iso.append(e0.elapsed_time(e1) * 1e3)
            del flush
            print(json.dumps({"config": name, "path": path, "chain": args.chain, "overlap": not args.no_overlap, "us_per_step": round(us, 3), "all": [round(t, 3) for t in times],
                              "frac": round(step_bytes / (us * 1e-6) / 6552.6e9, 3),
                              "isolated_us": round(float(np.median(iso)), 3),
                              "max_abs_diff_vs_first": diff, "launches": plan.stats()[0],
                              "path_bf16": sorted({d["path_bf16"] for d in desc}), "stream": desc[0].get("stream")}), flush=True)
            del g, plan


if __name__ == "__main__":
    main()
