#!/usr/bin/env python3
"""Per-CTA phase timeline of the fused bypass kernel (debug tracing).

    python tools/profile_trace.py --config cfg2 [--sm100 128,8,128,0]
Prints, per event, min / median / max over CTAs of (t_event - t_kernel_start) in us.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

EVENTS = ["start", "cluster_synced", "prod_shrink_issued", "mma_first_full", "mma_shrink_done",
          "epi_shrink_full", "epi_partials_sent", "owner_red_full", "owner_bcast_done", "mma_mid_full",
          "mma_expand_issued", "epi_first_acc", "epi_done", "end"]
# slots 14..30 are kernel specific (see the TRACE calls in kernels.cu)
EVENTS += [f"slot{_c}" for _c in range(14, 31)]
NEV = 32


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--sm100", default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ghz", type=float, default=1.92, help="SM clock for cycle -> ns")
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
    table = None
    if args.sm100:
        lc = tuple(int(v) for v in args.sm100.split(","))
        table = atmm.TilingTable()
        for m in sorted(set(w.lengths.values())):
            for r in set(w.ranks.values()):
                table.insert(atmm.m_bucket_of(m), w.d_in, r, (128, 128, 256, 128, 16, 64), 1, sm100=lc)
    plan = atmm.BypassPlan(reg, w.assignment, table)
    launches, tiles, ctas = plan.stats()
    x = torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y = torch.zeros(w.tokens, w.d_out, dtype=torch.bfloat16, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    tr = torch.zeros(ctas * NEV, dtype=torch.int64, device="cuda")
    plan.apply(x, y)
    torch.cuda.synchronize()
    print(f"{args.config}: launches={launches} tiles={tiles} ctas={ctas} sm100={args.sm100} groups={plan.describe()}")
    for rep in range(args.reps):
        flush.fill_(rep)
        tr.zero_()
        torch.cuda.synchronize()
        lib.atmm_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.apply(x, y)
        e1.record()
        torch.cuda.synchronize()
        lib.atmm_debug_set_trace(None)
        raw = tr.cpu().numpy().reshape(ctas, NEV).astype(np.float64)
        # events are clock64 cycles; anchor each CTA with its globaltimer (slot 31)
        ghz = args.ghz
        t = np.where(raw > 0, (raw - raw[:, :1]) / ghz + raw[:, NEV - 1:NEV], 0.0)
        t[:, NEV - 1] = 0
        t0 = t[:, 0][t[:, 0] > 0].min()
        print(f"rep {rep}: event-timed kernel {e0.elapsed_time(e1) * 1e3:.1f} us; "
              f"CTA start spread {(t[:, 0].max() - t0) / 1e3:.2f} us")
        own = np.where(raw > 0, (raw - raw[:, :1]) / ghz, np.nan)  # cycle-exact, per CTA
        for ev in range(min(NEV - 1, len(EVENTS))):
            col = t[:, ev]
            sel = col > 0
            col = col[sel]
            if col.size == 0:
                continue
            o = own[sel, ev] / 1e3
            rel = (col - t0) / 1e3
            print(f"   {ev:2d} {EVENTS[ev]:<20} n={col.size:4d}  min {rel.min():7.2f}  med {np.median(rel):7.2f}  "
                  f"max {rel.max():7.2f} us | own-clock med {np.nanmedian(o):7.3f}")


if __name__ == "__main__":
    main()
