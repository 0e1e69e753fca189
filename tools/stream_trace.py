#!/usr/bin/env python3
"""Per-CTA %globaltimer timeline of one atmm_stream_kernel launch (debug).

    python tools/stream_trace.py --config cfg2
Prints, per event, min / median / max over CTAs of (t_event - min start) in us.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

EVENTS = {0: "start", 6: "mma_first_shrink_full", 7: "mma_shrink_issued", 1: "sload_issued_all",
          3: "epi_partials_published", 9: "eload_after_wait", 2: "eload_issued_all", 4: "epi_first_tile_ready",
          8: "epi_first_mid_written", 11: "mma_first_expand", 10: "epi_first_unit_done", 5: "epi_done"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--warm", type=int, default=3)
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
    launch = list(atmm.heuristic_launch(128, w.d_in, 16, w.d_out))
    launch[4] = 4
    plan = atmm.BypassPlan(reg, w.assignment, launch=launch)
    x = torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y = torch.empty(w.tokens, w.d_out, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    for _ in range(args.warm):
        plan.apply(x, y)
    tr = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for rep in range(2):
        flush.fill_(rep)
        torch.cuda.synchronize()
        tr.zero_()
        lib.atmm_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
        plan.apply(x, y)
        torch.cuda.synchronize()
        lib.atmm_debug_set_trace(ctypes.c_void_p(0))
        t = tr.view(148, 32).cpu().numpy().astype(np.int64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        print(f"== {args.config} rep {rep}: stream kernel, {plan.describe()[0]['stream']}")
        for ev, name in EVENTS.items():
            v = t[:, ev]
            v = v[v > 0]
            if v.size == 0:
                continue
            d = (v - t0) / 1e3
            print(f"  {name:26s} n={v.size:4d} min {d.min():7.2f}  med {np.median(d):7.2f}  max {d.max():7.2f} us")


if __name__ == "__main__":
    main()
