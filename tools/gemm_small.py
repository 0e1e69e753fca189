#!/usr/bin/env python3
"""Small-m GEMM tile sweep (the base GEMM of the small-batch layer forward):
device time per call from a CUDA graph of 20 calls over 8 rotating W buffers
(256 MiB > L2), atmm_gemm tile options vs cuBLAS (torch.matmul).

    python tools/gemm_small.py [--m 16,64,128,256,512] [--k 4096] [--n 4096]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_00915_b200 as atmm  # noqa: E402

OPTS = [None, {"bn": 64, "kz": 1, "pair": 0}, {"bn": 64, "kz": 2, "pair": 0}, {"bn": 64, "kz": 4, "pair": 0},
        {"bn": 64, "mc": 2, "pair": 0}, {"bn": 64, "mc": 4, "pair": 0}, {"bn": 128, "kz": 2, "pair": 0},
        {"bn": 128, "mc": 4, "pair": 0}]


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", default="16,64,128,256,512")
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    args = ap.parse_args()
    k, n = args.k, args.n
    ws = [torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k**0.5 for _ in range(8)]
    for m in [int(v) for v in args.m.split(",")]:
        a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        ref = (a.double() @ ws[0].double())
        row = {"m": m, "k": k, "n": n, "cublas_us": round(graph_time(lambda i: torch.matmul(a, ws[i % 8], out=c)), 2)}
        for o in OPTS:
            key = "auto" if o is None else ",".join(f"{kk}{vv}" for kk, vv in o.items())
            try:
                row[key] = round(graph_time(lambda i: atmm.gemm(a, ws[i % 8], out=c, opts=o)), 2)
                got = atmm.gemm(a, ws[0], opts=o).double()
                err = float((got - ref).abs().max() / max(1.0, float(ref.abs().max())))
                if err > 1e-2:
                    row[key + "_err"] = err
            except Exception as e:  # noqa: BLE001
                row[key] = f"ERR {type(e).__name__}: {str(e)[:60]}"
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
