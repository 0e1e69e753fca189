"""atmm_gemm vs cuBLAS (torch.matmul) on bf16 shapes: TFLOP/s, CUDA events."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_00915_b200 as atmm  # noqa: E402


def timeit(fn, iters=50):
    for _ in range(min(5, iters)):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


SHAPES = [(16, 4096, 4096), (512, 4096, 4096), (1024, 4096, 4096), (2048, 4096, 4096), (4096, 4096, 4096),
          (8192, 8192, 8192), (16384, 4096, 4096)]


def main():
    for m, k, n in SHAPES:
        a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k**0.5
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        t_ours = timeit(lambda: atmm.gemm(a, b, out=c))
        t_cub = timeit(lambda: torch.matmul(a, b, out=c))
        err = (atmm.gemm(a, b).float() - torch.matmul(a, b).float()).abs().max().item()
        fl = 2.0 * m * k * n
        print(json.dumps({"m": m, "k": k, "n": n, "atmm_ms": round(t_ours, 4), "cublas_ms": round(t_cub, 4),
                          "atmm_tflops": round(fl / t_ours / 1e9, 1), "cublas_tflops": round(fl / t_cub / 1e9, 1),
                          "max_diff": err}))


if __name__ == "__main__":
    main()
