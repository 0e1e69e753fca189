#!/usr/bin/env python3
"""One small launch of every sm_100a kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [--only a2a,split]

Kernels: atmm_bypass_a2a_kernel, atmm_shrink_kernel + atmm_expand_kernel,
atmm_bypass_kernel (general fused), atmm_stream_kernel, atmm_merge_tma_kernel,
fwd_shrink_kernel + fwd_gemm_kernel (layer forward), atmm_gemm (1-SM, split-K,
2-SM pair).  Each result is checked against an fp64 product so a sanitizer
run is also a parity run.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PATHS = {"a2a": 1, "split": 2, "fused": 3, "stream": 4}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="a2a,split,fused,stream,overlap,chunks,merge,forward,gemm")
    ap.add_argument("--small", action="store_true", help="fewer rows (racecheck is slow)")
    args = ap.parse_args()
    only = set(args.only.split(","))
    import torch

    import paper_2411_00915_b200 as atmm

    rng = np.random.default_rng(0)
    d_in, d_out = 520, 392  # K tail (d_in % 64 != 0) and a partial last expand item
    ranks = {1: 16, 2: 32, 3: 64}
    lens = {1: 20, 2: 9, 3: 40} if args.small else {1: 40, 2: 17, 3: 130}
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    facs = {}
    for a, r in ranks.items():
        s = 1.0 / np.sqrt(r)
        facs[a] = (rng.uniform(-s, s, (d_in, r)).astype(np.float32), rng.uniform(-s, s, (r, d_out)).astype(np.float32))
        reg.put(a, facs[a][0], facs[a][1])
    asg = np.concatenate([np.full(n, a, np.int32) for a, n in lens.items()])
    asg = asg[rng.permutation(asg.size)]
    x = torch.empty(asg.size, d_in, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    xf = x.float().cpu().numpy().astype(np.float64)

    def want_bypass(y0):
        out = y0.astype(np.float64).copy()
        for i, a in enumerate(asg):
            d, u = facs[int(a)]
            dd = d.astype(np.float64)
            uu = u.astype(np.float64)
            out[i] += (xf[i] @ dd) @ uu
        return out

    for name, code in PATHS.items():
        if name not in only:
            continue
        for ydt in (torch.bfloat16, torch.float32):
            t = atmm.TilingTable()
            for a, r in ranks.items():
                launch = list(atmm.heuristic_launch(lens[a], d_in, r, d_out))
                launch[4] = code
                t.insert(atmm.m_bucket_of(lens[a]), d_in, r, (128, 128, 256, 128, 16, 64), 1, sm100=launch)
            plan = atmm.BypassPlan(reg, asg, t)
            y = torch.empty(asg.size, d_out, dtype=ydt, device="cuda").uniform_(-1, 1)
            y0 = y.float().cpu().numpy()
            for _ in range(2):  # the second launch reuses the per-stream scratch (split / stream counters)
                yy = y.clone()
                plan.apply(x, yy)
            torch.cuda.synchronize()
            err = float(np.max(np.abs(yy.float().cpu().numpy() - want_bypass(y0))))
            print(f"{name:7s} {str(ydt):15s} paths={sorted({g['path_bf16'] for g in plan.describe()})} max|err|={err:.3e}",
                  flush=True)
    if "overlap" in only:
        # consecutive independent applies on one stream: the later ones load
        # X / Y under their predecessor (dependency elision), then a dependent
        # one (X = the previous Y) that must wait
        t = atmm.TilingTable()
        for a, r in ranks.items():
            launch = list(atmm.heuristic_launch(lens[a], d_in, r, d_out))
            launch[4] = PATHS["a2a"]
            t.insert(atmm.m_bucket_of(lens[a]), d_in, r, (128, 128, 256, 128, 16, 64), 1, sm100=launch)
        plan = atmm.BypassPlan(reg, asg, t)
        ys = [torch.empty(asg.size, d_out, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1) for _ in range(3)]
        y0 = [y.float().cpu().numpy() for y in ys]
        before = atmm.overlap_stats()
        s_ = torch.cuda.Stream()
        with torch.cuda.stream(s_):
            for y in ys:
                plan.apply(x, y, stream=s_)
        s_.synchronize()
        after = atmm.overlap_stats()
        err = max(float(np.max(np.abs(y.float().cpu().numpy() - want_bypass(v)))) for y, v in zip(ys, y0))
        print(f"overlap early={after[1] - before[1]} of {after[0] - before[0]} max|err|={err:.3e}", flush=True)
    if "chunks" in only:
        rc = atmm.AdapterRegistry(1, d_in, d_out)
        s = 1.0 / np.sqrt(200)
        dn, up = rng.uniform(-s, s, (d_in, 200)).astype(np.float32), rng.uniform(-s, s, (200, d_out)).astype(np.float32)
        rc.put(7, dn, up)
        pl = atmm.BypassPlan(rc, np.full(48, 7, np.int32))
        xc = x[:48].contiguous()
        y = torch.zeros(48, d_out, dtype=torch.float32, device="cuda")
        pl.apply(xc, y)
        torch.cuda.synchronize()
        ref = (xc.double().cpu().numpy() @ dn.astype(np.float64)) @ up.astype(np.float64)
        print(f"chunks  passes={len({g['pass'] for g in pl.describe()})} max|err|={float(np.max(np.abs(y.cpu().numpy() - ref))):.3e}",
              flush=True)
    if "merge" in only:
        for wdt in (torch.bfloat16, torch.float32):
            W = torch.empty(d_in, d_out, dtype=wdt, device="cuda").uniform_(-0.05, 0.05)
            W0 = W.float().cpu().numpy().astype(np.float64)
            atmm.merge_into(reg, 3, 0, W, sign=1.0)
            torch.cuda.synchronize()
            d, u = facs[3]
            err = float(np.max(np.abs(W.float().cpu().numpy() - (W0 + d.astype(np.float64) @ u.astype(np.float64)))))
            print(f"merge   {str(wdt):15s} max|err|={err:.3e}", flush=True)
    if "forward" in only:
        sq = atmm.AdapterRegistry(2, d_in, d_in)
        for a, r in ranks.items():
            s = 1.0 / np.sqrt(r)
            sq.put(a, rng.uniform(-s, s, (2, d_in, r)).astype(np.float32), rng.uniform(-s, s, (2, r, d_in)).astype(np.float32))
        Wf = (torch.rand(2, d_in, d_in, device="cuda") * 2 - 1).mul_(1 / np.sqrt(d_in)).to(torch.bfloat16)
        fw = atmm.LayerForward(atmm.BypassPlan(sq, asg))
        out = torch.empty_like(x)
        fw.run(Wf, x, out)
        torch.cuda.synchronize()
        print(f"forward finite={bool(torch.isfinite(out.float()).all())}", flush=True)
    if "gemm" in only:
        for m in (64, 300):
            a = torch.empty(m, 512, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
            b = torch.empty(512, 640, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
            c = atmm.gemm(a, b, out_dtype=torch.float32)
            torch.cuda.synchronize()
            ref = a.double() @ b.double()
            print(f"gemm    m={m} max|err|={float((c.double() - ref).abs().max()):.3e}", flush=True)


if __name__ == "__main__":
    main()
