#!/usr/bin/env python3
"""Steady-state per-step timeline of the bypass kernel inside a K-step CUDA
graph (the bench's timed region), from per-CTA %globaltimer / clock64 traces.

Each captured step gets its own trace buffer (the pointer is baked into the
launch at capture time), X / Y rotate over > 2 x L2 like bench.py.  Prints,
per step, the phase times relative to the END of the previous step's grid
(last CTA exit): how long the wait on the previous grid takes to return,
when X lands, when the exchange completes, when Y is written -- i.e. where
the per-step period goes once consecutive steps overlap through PDL.

    python tools/step_timeline.py --config cfg2 [--steps 12] [--x-ready] [--out gpurun_out/timeline.json]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

NEV = 32
L2_BYTES = 126 * 1024 * 1024
# a2a kernel events (kernels.cu TRACE calls)
A2A = {0: "start", 1: "setup_done", 15: "x_wait_returned", 16: "y_wait_returned", 2: "x_gathers_issued", 3: "first_x_stage",
       22: "trigger_wait_returned", 4: "shrink_mma_done", 5: "partials_in_tmem", 23: "tmem_loaded", 17: "partials_in_smem",
       18: "proxy_fenced", 19: "cluster_waited", 20: "bar_synced", 6: "partials_pushed", 7: "peers_partials_in",
       8: "mid_written", 9: "expand_start", 11: "expand_acc_ready", 14: "y_staged", 12: "y_written", 13: "end", 24: "exit"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--ghz", type=float, default=1.965, help="SM clock for clock64 -> ns")
    ap.add_argument("--x-ready", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_2411_00915_b200 as atmm
    from paper_2411_00915_b200._lib import lib
    from paper_2411_00915_b200.workloads import bypass_config

    lib.atmm_debug_set_trace.argtypes = [ctypes.c_void_p]
    w = bypass_config(args.config)
    step_bytes = w.bytes(2)
    nbuf = min(64, max(2, int(np.ceil(2.5 * L2_BYTES / step_bytes))))
    rng = np.random.default_rng(0)
    reg = atmm.AdapterRegistry(nbuf, w.d_in, w.d_out)
    for a, r in w.ranks.items():
        s = 1.0 / np.sqrt(r)
        reg.put(a, rng.uniform(-s, s, (nbuf, w.d_in, r)).astype(np.float32),
                rng.uniform(-s, s, (nbuf, r, w.d_out)).astype(np.float32))
    plan = atmm.BypassPlan(reg, w.assignment)
    if args.x_ready:
        plan.set_x_ready(True)
    launches, tiles, ctas = plan.stats()
    dev = torch.device("cuda", 0)
    xs = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device=dev).uniform_(-1, 1) for _ in range(nbuf)]
    ys = [torch.empty(w.tokens, w.d_out, dtype=torch.bfloat16, device=dev).uniform_(-1, 1) for _ in range(nbuf)]
    K = args.steps
    tr = torch.zeros(K, ctas * NEV, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for i in range(3):
            plan.apply(xs[i % nbuf], ys[i % nbuf], layer=i % nbuf, stream=stream)
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
        for i in range(K):
            lib.atmm_debug_set_trace(ctypes.c_void_p(tr[i].data_ptr()))
            plan.apply(xs[i % nbuf], ys[i % nbuf], layer=i % nbuf, stream=stream)
    lib.atmm_debug_set_trace(None)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    tr.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    total_us = e0.elapsed_time(e1) * 1e3
    raw = tr.cpu().numpy().reshape(K, ctas, NEV).astype(np.float64)
    # absolute ns: globaltimer of event 0 (slot 31) + clock64 deltas
    t = np.where(raw > 0, (raw - raw[:, :, :1]) / args.ghz + raw[:, :, NEV - 1:NEV], np.nan)
    t[:, :, NEV - 1] = np.nan
    t0 = np.nanmin(t[:, :, 0])
    t = (t - t0) / 1e3  # us from the first CTA start of step 0
    ends = np.nanmax(t[:, :, 24], axis=1)  # the last CTA past its final cluster barrier
    starts = np.nanmin(t[:, :, 0], axis=1)
    rows = []
    print(f"{args.config}: {K} steps in one graph, {total_us / K:.2f} us/step (events), ctas/step={ctas}, "
          f"x_ready={args.x_ready}")
    print("step  first_start  last_end  period | phase medians rel. to previous grid end (us)")
    for i in range(K):
        prev_end = ends[i - 1] if i > 0 else np.nan
        rec = {"step": i, "first_cta_start_us": float(starts[i]), "last_cta_end_us": float(ends[i]),
               "period_us": float(ends[i] - prev_end) if i > 0 else None, "phases": {}}
        parts = []
        for ev, name in A2A.items():
            col = t[i, :, ev]
            if np.all(np.isnan(col)):
                continue
            rel = col - (prev_end if i > 0 else starts[i])
            rec["phases"][name] = {"min": float(np.nanmin(rel)), "med": float(np.nanmedian(rel)),
                                   "max": float(np.nanmax(rel))}
            parts.append(f"{name}={np.nanmedian(rel):.2f}")
        rows.append(rec)
        per = f"{ends[i] - prev_end:6.2f}" if i > 0 else "   -  "
        print(f"{i:4d} {starts[i]:10.2f} {ends[i]:9.2f} {per} | " + " ".join(parts))
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"config": args.config, "steps": K, "us_per_step_events": total_us / K, "ctas": ctas,
                       "x_ready": args.x_ready, "reference_point": "previous step's last CTA exit (event 24, after the final cluster barrier)",
                       "records": rows}, f, indent=1)


if __name__ == "__main__":
    main()
