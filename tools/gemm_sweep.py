"""atmm_gemm tile-config sweep (ATMM_FWD_PAIR / BN / KZ) on chosen shapes."""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_00915_b200 as atmm  # noqa: E402
from tools.gemm_bench import timeit  # noqa: E402

ITERS = int(os.environ.get("GEMM_SWEEP_ITERS", "200"))


def graph_time(fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph (no host
    launch overhead), replayed ITERS / reps times."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    return timeit(g.replay, max(1, ITERS // reps)) / reps


def main():
    shapes = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[1:] or ["512x4096x4096", "256x4096x4096"])]
    for m, k, n in shapes:
        a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k**0.5
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        t_cub = graph_time(lambda: torch.matmul(a, b, out=c))
        want = torch.matmul(a, b).float()
        for pair, bn, kz, mc in itertools.product(["0", "1"], ["128", "256"], ["1", "2", "4"], ["1", "2", "4"]):
            if (pair == "1" and (kz != "1" or mc != "1")) or (kz != "1" and mc != "1"):
                continue
            os.environ.update(ATMM_FWD_PAIR=pair, ATMM_FWD_BN=bn, ATMM_FWD_KZ=kz, ATMM_GEMM_MC=mc)
            t = graph_time(lambda: atmm.gemm(a, b, out=c))
            err = (c.float() - want).abs().max().item()
            print(json.dumps({"shape": [m, k, n], "pair": pair, "bn": bn, "kz": kz, "mc": mc, "us": round(t * 1e3, 2),
                              "cublas_us": round(t_cub * 1e3, 2), "err": err}))


if __name__ == "__main__":
    main()
