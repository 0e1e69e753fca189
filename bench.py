#!/usr/bin/env python3
"""bench.py -- ATMM batched-LoRA benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg1|cfg3|cfg5|cfg4|paper_in1|paper_in2]

A step is ONE fused bypass pass  Y[rows] += (X[rows] . down_a) . up_a  over
one batch (default cfg2 = BASELINE.json configs[1]: hidden 4096, rank 16,
16 adapters, 512 tokens, bf16, 1 x B200).  The workload fits in L2, so steps
rotate over 32 layer buffer sets (X, Y and adapter factors per layer,
> 2 x L2 in total).  K steps are captured in one CUDA graph and replayed
inside the timed region (barrier + synchronize on both sides, CUDA events,
max over ranks).  Under torchrun each rank runs its own batch of requests
(request sharding, no collective on the data path): scaling = weak.

One JSON line on rank 0 with value (TFLOP/s, whole job), ms_per_step, the
dominant kernel's roofline, the CPU baseline (the reference compiled from
its own headers, oracle/_ref, on a bounded sample), the end-to-end number
through the C ABI with pinned host buffers, and SM clocks sampled during
the run.  --impl reference times the reference CPU implementation instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ATMM batched-LoRA TFLOP/s and µs/batch at Qwen-VL-7B shapes vs CPU ref"
L2_BYTES = 126 * 1024 * 1024
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (GB/s)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--cpu-sample-s", type=float, default=10.0, help="bounded CPU baseline sample (seconds)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--soak-s", type=float, default=1.0, help="load before the timed region while clocks are sampled")
    ap.add_argument("--group", type=int, default=3, help="extra measurement: steps per grouped launch (1 = off)")
    ap.add_argument("--no-forward", action="store_true", help="skip the layer-forward side measurement")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: split the workload itself over the N ranks (default: weak, one batch per GPU)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


def committed_ncu(config: str) -> dict:
    """The committed ncu capture of this config's kernel(s) (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_bypass_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(config, {})
    return {}


def committed_traffic(config: str):
    """dram bytes per launch of the bypass kernel from the committed ncu capture."""
    return committed_ncu(config).get("dram_bytes_per_launch")


def isolated_frac(config: str, step_bytes: int, peak: float):
    """Roofline fraction of ONE isolated launch (ncu: cold cache, serialised,
    no overlap with the neighbouring steps) beside the pipelined `frac`."""
    us = committed_ncu(config).get("duration_us")
    return (step_bytes / (us * 1e-6) / 1e9 / peak, us) if us else (None, None)


# ------------------------------------------------------------ clocks ------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() in ("active", "0x1", "1"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "window": "soak + timed region"}


# ------------------------------------------------------ distributed -------
DIST_BACKEND = os.environ.get("ATMM_BENCH_DIST", "nccl")  # "gloo": multi-rank smoke test on one GPU


def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if n_gpus > 1 and world == 1:
        raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch

        if DIST_BACKEND == "gloo":  # every rank on the one visible GPU (code-path test, not a measurement)
            local = 0
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cpu" if DIST_BACKEND == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# -------------------------------------------------- reference (CPU) -------
def reference_batch_fn(w, seed: int):
    """Returns (fn, flops): fn() runs the reference's run_bypass (batch.hpp:48)
    on one fp32 batch."""
    from oracle.oracle import Reference

    ref = Reference()
    rng = np.random.default_rng(seed)
    adapters = {}
    for a, r in w.ranks.items():
        s = 1.0 / np.sqrt(r)
        adapters[a] = (rng.uniform(-s, s, (w.d_in, r)).astype(np.float32),
                       rng.uniform(-s, s, (r, w.d_out)).astype(np.float32))
    ctx = ref.ctx(w.d_in, adapters)
    x = rng.uniform(-1, 1, (w.tokens, w.d_in)).astype(np.float32)
    a = np.ascontiguousarray(w.assignment, np.int32)

    def fn():
        return ctx.run_bypass(x, a)  # batch.hpp:48 run_bypass: a fresh n x d_out bypass

    return fn, w.flops()


def run_reference_parallel(w, threads: int, seconds: float = None, steps: int = None):
    """`threads` independent request batches through the reference on as
    many host cores (ctypes releases the GIL).  Returns (wall seconds, batches)."""
    fns = [reference_batch_fn(w, 100 + t)[0] for t in range(threads)]
    counts = [0] * threads
    stop = threading.Event()

    def worker(i):
        if steps is not None:
            for _ in range(steps):
                fns[i]()
                counts[i] += 1
        else:
            while not stop.is_set():
                fns[i]()
                counts[i] += 1

    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    if steps is None:
        time.sleep(seconds)
        stop.set()
    for t in ths:
        t.join()
    return time.perf_counter() - t0, sum(counts)


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_config(w, world: int) -> dict:
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": w.name, "d_in": w.d_in, "d_out": w.d_out, "tokens": w.tokens, "adapters": len(w.ranks),
            "ranks": sorted(set(w.ranks.values())), "segment_rows": sorted(set(w.lengths.values()))[:4],
            "parallelism": f"request-sharded x{world} (no collective)"}


def merge_config(mw, world: int) -> dict:
    return {"workload": "cfg4", "d_in": mw.d_in, "d_out": mw.d_out, "rank": mw.rank, "layers": mw.layers,
            "w_dtype": "bf16", "parallelism": f"layer-sharded x{world} (no collective)"}


def reference_one_thread_rate(w, seconds: float = 2.0) -> float:
    """The reference's run_bypass on ONE host thread (LORASERVE_THREADS=1,
    its default), TFLOP/s over a bounded sample."""
    os.environ["LORASERVE_THREADS"] = "1"
    el, batches = run_reference_parallel(w, 1, seconds=seconds)
    return w.flops() * batches / el / 1e12


def reference_merge_rate(mw, threads: int, layers: int = 1):
    """The reference's merge of ONE cfg4 layer: delta_w_into (its tiled ATMM,
    model.hpp:120-125) + add_inplace (model.hpp:157-158) through
    oracle/_ref's ref_merge_rect, LORASERVE_THREADS=threads (atmm.hpp:126-141
    splits the 4096 output rows over that many jthreads).  Returns
    (seconds per layer, TFLOP/s)."""
    from oracle.oracle import Reference

    ref = Reference()
    os.environ["LORASERVE_THREADS"] = str(threads)
    rng = np.random.default_rng(21)
    s = 1.0 / np.sqrt(mw.rank)
    down = rng.uniform(-s, s, (mw.d_in, mw.rank)).astype(np.float32)
    up = rng.uniform(-s, s, (mw.rank, mw.d_out)).astype(np.float32)
    W = rng.uniform(-1 / np.sqrt(mw.d_in), 1 / np.sqrt(mw.d_in), (mw.d_in, mw.d_out)).astype(np.float32)
    ref.merge_rect(W, down, up, 1)  # warm-up (page faults, allocator)
    t0 = time.perf_counter()
    for i in range(layers):
        ref.merge_rect(W, down, up, -1 if i % 2 else 1)
    el = (time.perf_counter() - t0) / layers
    per_layer_flops = 2 * mw.d_in * mw.d_out * mw.rank + mw.d_in * mw.d_out
    return el, per_layer_flops / el / 1e12


def impl_reference(args, w):
    rank, world, _ = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), 0
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    threads = cpu_threads()
    for _ in range(max(args.warmup, 1)):
        run_reference_parallel(w, threads, steps=1)
    elapsed, batches = run_reference_parallel(w, threads, steps=args.steps)
    flops = w.flops() * batches
    value = flops / elapsed / 1e12
    cfg = bench_config(w, world)
    sample = (f"{args.steps} steps x {threads} concurrent {w.name} batches (one per host thread) through the "
              f"reference's run_bypass (batch.hpp:48), fp32, oracle/_ref built from the reference headers")
    one = reference_one_thread_rate(w)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model(), "value_1thread": one},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def impl_reference_merge(args):
    """cfg4 reference arm: the reference's merge (delta_w_into + add_inplace)
    of one 4096 x 11008 rank-64 layer per step, all host threads; the rate
    is comparable with the GPU arm's all-32-layer TFLOP/s."""
    from paper_2411_00915_b200.workloads import MergeWorkload

    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    mw = MergeWorkload()
    threads = cpu_threads()
    for _ in range(max(args.warmup, 1)):
        reference_merge_rate(mw, threads, 1)
    el, rate = reference_merge_rate(mw, threads, args.steps)
    _, one = reference_merge_rate(mw, 1, 1)
    sample = (f"{args.steps} steps, each ONE cfg4 layer (4096 x 11008, r64, fp32) through the reference's "
              f"delta_w_into + add_inplace (model.hpp:120-125,157-158) with LORASERVE_THREADS={threads}; "
              f"ms_per_step projects the 32-layer merge")
    line = {
        "impl": "reference", "metric": "ATMM merge/unmerge W +- s.down.up, all 32 layers (mode switch) TFLOP/s",
        "value": rate, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el * mw.layers * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": merge_config(mw, world),
        "cpu_baseline": {"value": rate, "unit": "TFLOP/s", "cores": threads, "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model(), "value_1thread": one},
        "e2e": {"value": rate, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------- ours (GPU) ------
def reference_forward_rate(w, seconds: float):
    """The reference's forward_unmerged (model.hpp:216-246, fp32, its tiled
    ATMM) on a bounded row sample of this workload, one layer, one sample per
    host thread in parallel: TFLOP/s of 2 n d^2 + bypass FLOPs."""
    from oracle.oracle import Reference

    ref = Reference()
    d, rows = w.d_in, 16
    threads = cpu_threads()
    rng = np.random.default_rng(9)
    W = rng.uniform(-1 / np.sqrt(d), 1 / np.sqrt(d), (1, d, d)).astype(np.float32)
    ads = {}
    for a, r in w.ranks.items():
        s = 1.0 / np.sqrt(r)
        ads[a] = (rng.uniform(-s, s, (1, d, r)).astype(np.float32), rng.uniform(-s, s, (1, r, d)).astype(np.float32))
    asg = np.ascontiguousarray(w.assignment[:rows], np.int32)
    x = rng.uniform(-1, 1, (rows, d)).astype(np.float32)
    sub = {a: ads[a] for a in set(asg.tolist())}
    flops = 2 * rows * d * d + sum(4 * d * w.ranks[int(a)] for a in asg)
    ref.forward(x, W, "unmerged", asg, sub)  # warm-up
    counts = [0] * threads
    stop = threading.Event()

    def worker(i):
        while not stop.is_set():
            ref.forward(x, W, "unmerged", asg, sub)
            counts[i] += 1

    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    time.sleep(seconds)
    stop.set()
    for t in ths:
        t.join()
    el = time.perf_counter() - t0
    return {"tflops": flops * sum(counts) / el / 1e12, "cores": threads, "kind": "reference",
            "sample": f"{sum(counts)} calls of forward_unmerged on {rows} rows x 1 layer (d {d}) in {el:.1f} s, "
                      f"one per host thread, oracle/_ref built from the reference headers"}


def measure_forward(atmm, plan, w, x, stream, reps=10, num_layers=2, cpu_sample_s=0.0):
    """Side measurement (not the headline): the model's layer forward
    tanh(x W_l + bypass_l(x)) (model.hpp:216-246) on this batch through
    LayerForward (bypass fused into the base GEMM as extra K blocks), beside
    the unfused composition cuBLAS x @ W + our bypass kernel + tanh, and
    cuBLAS alone.  CUDA graph of `reps` forwards, per-layer us."""
    import torch

    d = w.d_in
    W = (torch.rand(num_layers, d, d, device=x.device) * 2 - 1).mul_(1.0 / np.sqrt(d)).to(torch.bfloat16)
    fw = atmm.LayerForward(plan)
    out = torch.empty_like(x)
    bufs = [torch.empty_like(x) for _ in range(2)]

    def fused():
        fw.run(W, x, out, stream=stream)

    def unfused():
        cur = x
        for l in range(num_layers):
            y = bufs[l % 2]
            torch.mm(cur, W[l], out=y)
            plan.apply(cur, y, layer=l, stream=stream)
            torch.tanh_(y)
            cur = y

    def cublas():
        cur = x
        for l in range(num_layers):
            torch.mm(cur, W[l], out=bufs[l % 2])
            cur = bufs[l % 2]

    def per_layer_us(fn):
        with torch.cuda.stream(stream):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
            for _ in range(reps):
                fn()
        best = float("inf")
        with torch.cuda.stream(stream):
            g.replay()
            torch.cuda.synchronize()
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e3 / (reps * num_layers))
        return best

    t_f, t_u, t_c = per_layer_us(fused), per_layer_us(unfused), per_layer_us(cublas)
    flops = 2 * w.tokens * d * d + w.flops()
    cpu_ref = None
    if cpu_sample_s > 0:
        try:
            cpu_ref = reference_forward_rate(w, cpu_sample_s)
        except FileNotFoundError as e:
            cpu_ref = {"unavailable": str(e)}
    peak = measured_bf16_peak()
    st = fw.stats()
    return {"us_per_layer": t_f, "tflops": flops / (t_f * 1e-6) / 1e12,
            "roofline": {"bound": "tensor", "peak": peak, "unit": "TFLOP/s",
                         "frac": flops / (t_f * 1e-6) / 1e12 / peak if peak else None},
            "unfused_us_per_layer": t_u, "cublas_mm_only_us_per_layer": t_c, "cpu_reference": cpu_ref,
            "layers": num_layers, "launches_per_layer": 2, "gemm_tile_n": st["bn"], "shrink_k_split": st["shrink_ks"],
            "note": "side measurement: tanh(x W + bypass) per layer, fused forward (fwd_shrink + fwd_gemm) vs "
                    "cuBLAS x@W + bypass kernel + tanh; W bf16 random, not the headline"}


def measured_bf16_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f).get("bf16_tflops") or 0) or None
    return 2250.0


def impl_ours_bypass(args, w):
    import torch

    rank, world, local = dist_setup(args.gpus)
    import paper_2411_00915_b200 as atmm

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    # Request sharding: the job's global batch is split by
    # whole segments over the ranks (LPT, every rank derives the same plan);
    # each rank holds only its shard's adapters and rows.  Weak scaling
    # (default): the global batch is N independent copies of the workload,
    # one per GPU.  --strong: the workload itself is split N ways.
    from paper_2411_00915_b200.sharding import ShardedBypass, replicate_batch, shard_flops
    from paper_2411_00915_b200.workloads import BypassWorkload

    if args.strong:
        glob, granks = w.assignment, dict(w.ranks)
    else:
        glob, granks = replicate_batch(w.assignment, w.ranks, world)
    # per-rank shard description (lw): rows, adapters and lengths of this rank
    from paper_2411_00915_b200.sharding import shard_batch

    shards = shard_batch(glob, granks, w.d_in, w.d_out, world)
    mine = shards[rank]
    ids, counts = np.unique(mine.assignment, return_counts=True)
    lw = BypassWorkload(w.name, w.d_in, w.d_out, int(mine.rows.size), {int(a): granks[int(a)] for a in ids},
                        {int(a): int(c) for a, c in zip(ids, counts)}, mine.assignment)
    job_flops = sum(shard_flops(sh, granks, w.d_in, w.d_out) for sh in shards)
    step_bytes = lw.bytes(2)
    layers = max(2, int(np.ceil(2.5 * L2_BYTES / step_bytes)))
    layers = min(layers, 64)

    def factors(a):  # every layer's factors of adapter a (same on every rank)
        rng = np.random.default_rng(1234 + a)
        r = granks[a]
        s = 1.0 / np.sqrt(r)
        return (rng.uniform(-s, s, (layers, w.d_in, r)).astype(np.float32),
                rng.uniform(-s, s, (layers, r, w.d_out)).astype(np.float32))

    sb = ShardedBypass(glob, granks, w.d_in, w.d_out, world, rank, factors, num_layers=layers, device=local)
    reg, plan = sb.registry, sb.plan
    w_job = w
    w = lw  # per-rank quantities below (tokens, bytes, flops of this rank's shard)
    launches_per_step, tiles, ctas = plan.stats()
    xs = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device=dev).uniform_(-1, 1) for _ in range(layers)]
    ys = [torch.empty(w.tokens, w.d_out, dtype=torch.bfloat16, device=dev).uniform_(-1, 1) for _ in range(layers)]
    stream = torch.cuda.Stream(device=dev)

    def step(i, s):
        l = i % layers
        plan.apply(xs[l], ys[l], layer=l, scale=1.0, stream=s)

    # warm-up (untimed), eager
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i, stream)
    torch.cuda.synchronize()

    # Capture exactly K steps into one graph.
    g = torch.cuda.CUDAGraph()
    ov0 = atmm.overlap_stats()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
        for i in range(args.steps):
            step(i, stream)
    ov1 = atmm.overlap_stats()
    overlap = {"a2a_launches": ov1[0] - ov0[0], "early_launches": ov1[1] - ov0[1],
               "rule": "an all-to-all launch loads X / Y under its predecessor only when the launcher proved the "
                       "predecessor (the one grid that can still run) touches disjoint bytes (include/atmm_b200.h "
                       "ATMM_PLAN_NO_OVERLAP)"}
    # Soak graph for clock steady state.
    soak_steps = min(args.steps, 4 * layers)
    gs = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gs, stream=stream, capture_error_mode="thread_local"):
        for i in range(soak_steps):
            step(i, stream)
    g.replay()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    t_end = time.perf_counter() + args.soak_s
    with torch.cuda.stream(stream):
        while time.perf_counter() < t_end:
            gs.replay()
            stream.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop()
    ms_local = e0.elapsed_time(e1)
    ms = max_over_ranks(ms_local, world)

    # ---- ATMM_PLAN_X_READY: the same K steps with X gathered before
    # griddepcontrol.wait (X is never written here; a bypass that follows the
    # base GEMM Y = X W may promise the same).  Side measurement ----
    x_ready = None
    plan.set_x_ready(True)
    gx = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gx, stream=stream, capture_error_mode="thread_local"):
        for i in range(args.steps):
            step(i, stream)
    plan.set_x_ready(False)
    gx.replay()
    torch.cuda.synchronize()
    x0 = torch.cuda.Event(enable_timing=True)
    x1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        x0.record(stream)
        gx.replay()
        x1.record(stream)
    torch.cuda.synchronize()
    xms = max_over_ranks(x0.elapsed_time(x1), world)
    x_ready = {"us_per_batch": xms * 1e3 / args.steps,
               "value": job_flops * args.steps / (xms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "roofline_frac": step_bytes / (xms * 1e-3 / args.steps) / 1e9 / measured_peaks()[0],
               "note": "same steps with atmm_plan_set_flags(ATMM_PLAN_X_READY): X gathered under the previous "
                       "launch's tail; not the headline"}

    # ---- dependent chain: step i+1 reads step i's output as its X (a layer
    # forward's data flow).  The launcher's hazard check then keeps the full
    # grid dependency (no X / Y loads under the predecessor): the number a
    # caller with strictly dependent steps sees.  Side measurement ----
    chain = None
    if w.d_in == w.d_out:
        gc = torch.cuda.CUDAGraph()
        early0 = atmm.overlap_stats()
        with torch.cuda.graph(gc, stream=stream, capture_error_mode="thread_local"):
            for i in range(args.steps):
                plan.apply(ys[i % layers], ys[(i + 1) % layers], layer=i % layers, scale=1.0, stream=stream)
        early1 = atmm.overlap_stats()
        gc.replay()
        torch.cuda.synchronize()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        barrier(world)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            c0.record(stream)
            gc.replay()
            c1.record(stream)
        torch.cuda.synchronize()
        cms = max_over_ranks(c0.elapsed_time(c1), world)
        chain = {"us_per_batch": cms * 1e3 / args.steps,
                 "value": job_flops * args.steps / (cms * 1e-3) / 1e12, "unit": "TFLOP/s",
                 "roofline_frac": step_bytes / (cms * 1e-3 / args.steps) / 1e9 / measured_peaks()[0],
                 "early_launches": early1[1] - early0[1],
                 "note": "X of step i+1 = Y of step i: every launch keeps the full grid dependency; not the headline"}

    # ---- single-launch latency: one eager call bracketed by
    # events on an idle GPU, median of 20 (includes the launch itself) ----
    single = []
    with torch.cuda.stream(stream):
        for i in range(20):
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a0.record(stream)
            step(i, stream)
            a1.record(stream)
            torch.cuda.synchronize()
            single.append(a0.elapsed_time(a1) * 1e3)
    single_launch_us = float(np.median(single))

    # ---- grouped launches: G consecutive independent steps (e.g. the q/k/v
    # projections of one decoder layer) as ONE launch (atmm_bypass_apply_group) ----
    grouped = None
    G = args.group
    if G > 1:
        gsteps = (args.steps // G) * G
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gg, stream=stream, capture_error_mode="thread_local"):
            for i0 in range(0, gsteps, G):
                ls = [(i0 + k) % layers for k in range(G)]
                plan.apply_group([xs[l] for l in ls], [ys[l] for l in ls], ls, stream=stream)
        gg.replay()
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        barrier(world)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            g0.record(stream)
            gg.replay()
            g1.record(stream)
        torch.cuda.synchronize()
        gms = max_over_ranks(g0.elapsed_time(g1), world)
        grouped = {"calls_per_launch": G, "us_per_batch": gms * 1e3 / gsteps,
                   "value": job_flops * gsteps / (gms * 1e-3) / 1e12, "unit": "TFLOP/s",
                   "roofline_frac": step_bytes / (gms * 1e-3 / gsteps) / 1e9 / measured_peaks()[0],
                   "note": "same steps, G independent (X, Y, layer) calls per launch; not the headline"}

    layer_fwd = None
    if not args.no_forward and w.d_in == w.d_out:
        layer_fwd = measure_forward(atmm, plan, w, xs[0], stream, reps=20, num_layers=min(4, layers),
                                    cpu_sample_s=0.0 if (args.no_cpu_baseline or world > 1 or rank != 0) else 3.0)

    flops_step = w.flops()
    value = job_flops * args.steps / (ms * 1e-3) / 1e12
    ms_per_step = ms / args.steps
    # The step is the hot path: one fused launch (all-to-all or general fused
    # kernel) or the split shrink + expand pair.  Achieved bandwidth = the
    # step's algorithmic bytes / the step's device time (all its launches).
    groups = plan.describe()
    paths = sorted({g.get("path_bf16", "fused") for g in groups})
    kernel_names = {"a2a": "atmm_bypass_a2a_kernel", "split": "atmm_shrink_kernel+atmm_expand_kernel",
                    "fused": "atmm_bypass_kernel"}
    kernel_us = ms_local * 1e3 / args.steps
    hbm_peak, peak_kind = measured_peaks()
    achieved_gbs = step_bytes / (kernel_us * 1e-6) / 1e9
    frac_iso, iso_us = isolated_frac(w.name, step_bytes, hbm_peak)

    # ---- end to end through the C ABI with pinned host buffers ----
    # run_bypass (batch.hpp:48) semantics, the reference's own call: every
    # step H2D of that step's X from pinned host memory, the bypass into a
    # fresh output, D2H of the output; independent batches pipelined over
    # three streams (atmm_run_bypass_host_bf16_pipelined).  The residual
    # form (Y in, Y += bypass, Y out) is reported beside it.
    e2e = None
    e2e_res = None
    e2e_rb = None
    if not args.no_e2e:
        # enough batches that pipeline fill / drain (3 slots) is amortised;
        # independent of --steps (the e2e leg is a few ms of PCIe traffic)
        e2e_steps = 128
        nbuf = 6
        xh = [torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16).uniform_(-1, 1).pin_memory() for _ in range(nbuf)]
        yh = [torch.zeros(w.tokens, w.d_out, dtype=torch.bfloat16).pin_memory() for _ in range(nbuf)]
        xs = [t.view(torch.int16).numpy().view(np.uint16) for t in xh]
        ys = [t.view(torch.int16).numpy().view(np.uint16) for t in yh]
        seq_x = [xs[i % nbuf] for i in range(e2e_steps)]
        seq_y = [ys[i % nbuf] for i in range(e2e_steps)]
        seq_l = [i % layers for i in range(e2e_steps)]

        def timed(fn):
            fn(seq_x[:3], seq_y[:3], seq_l[:3])  # warm-up
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(seq_x, seq_y, seq_l)
            torch.cuda.synchronize()
            return max_over_ranks(time.perf_counter() - t0, world)

        e2e_s = timed(lambda a, b, c: atmm.run_bypass_host_bf16_pipelined(plan, a, b, c))
        e2e = {"value": job_flops * e2e_steps / e2e_s / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(w.tokens * w.d_in * 2),
               "d2h_bytes_per_step": int(w.tokens * w.d_out * 2),
               "us_per_batch": e2e_s / e2e_steps * 1e6, "steps": e2e_steps,
               "path": "atmm_run_bypass_host_bf16_pipelined = run_bypass (batch.hpp:48) on pinned bf16 host "
                       "buffers: H2D X, fused kernel into a fresh output, D2H; 4 streams"}
        r_s = timed(lambda a, b, c: atmm.residual_host_bf16_pipelined(plan, a, b, c))
        e2e_res = {"value": job_flops * e2e_steps / r_s / 1e12, "unit": "TFLOP/s",
                   "h2d_bytes_per_step": int(w.tokens * (w.d_in + w.d_out) * 2),
                   "d2h_bytes_per_step": int(w.tokens * w.d_out * 2), "us_per_batch": r_s / e2e_steps * 1e6,
                   "path": "atmm_bypass_residual_host_bf16_pipelined: H2D X and Y, Y += bypass, D2H Y"}
        # the reference's own signature, one synchronous call per batch:
        # run_bypass(x, plan, adapters, layer, table) (batch.hpp:48) with fp32
        # host buffers, as include/loraserve_compat.hpp calls it
        xf32 = np.random.default_rng(9).uniform(-1, 1, (w.tokens, w.d_in)).astype(np.float32)
        for _ in range(3):
            atmm.run_bypass(reg, xf32, w.assignment, layer=0)
        torch.cuda.synchronize()
        calls = 30
        t0 = time.perf_counter()
        for i in range(calls):
            atmm.run_bypass(reg, xf32, w.assignment, layer=i % layers)
        rb_s = max_over_ranks(time.perf_counter() - t0, world)
        e2e_rb = {"value": job_flops * calls / rb_s / 1e12, "unit": "TFLOP/s",
                  "h2d_bytes_per_step": int(w.tokens * w.d_in * 4), "d2h_bytes_per_step": int(w.tokens * w.d_out * 4),
                  "us_per_batch": rb_s / calls * 1e6,
                  "path": "atmm_run_bypass_host = run_bypass (batch.hpp:48) signature: fp32 host x in, fresh fp32 "
                          "bypass out, one synchronous call per batch (plan cached, buffers reused)"}

    # ---- CPU baseline: the reference itself, bounded sample, rank 0, N=1 ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = cpu_threads()
            run_reference_parallel(w, threads, steps=1)
            el, batches = run_reference_parallel(w, threads, seconds=args.cpu_sample_s)
            cpu = {"value": w.flops() * batches / el / 1e12, "unit": "TFLOP/s", "cores": threads,
                   "kind": "reference",
                   "sample": f"{batches} {w.name} batches in {el:.1f} s, {threads} concurrent batches "
                             f"(one per host thread) through the reference run_bypass (batch.hpp:48, fp32), "
                             f"oracle/_ref built from the reference headers",
                   "cpu_model": cpu_model(), "value_1thread": reference_one_thread_rate(w)}
        except FileNotFoundError as e:
            cpu = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "us_per_batch": ms_per_step * 1e3,
            "single_launch_us": single_launch_us,
            "x_ready": x_ready,
            "dependent_chain": chain,
            "overlap": overlap,
            "config": bench_config(w_job, world),
            "sharding": {"mode": "strong" if args.strong else "weak", "global_tokens": int(len(glob)),
                         "global_adapters": len(granks), "rank0_tokens": int(w.tokens),
                         "rank0_adapters": len(w.ranks), "collective": None,
                         "launcher": "paper_2411_00915_b200.sharding.ShardedBypass (LPT over whole segments, "
                                     "atmm_shard_rows; only the shard's adapters resident)"},
            "timing": {"l2": f"inputs rotate over {layers} layer buffer sets ({layers * step_bytes / 2**20:.0f} MiB "
                             f"> 2x L2); K steps in one CUDA graph, CUDA events on the launch stream"},
            "plan": {"launches_per_step": launches_per_step, "tiles": tiles, "ctas": ctas,
                     "launch_groups": plan.describe()},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved_gbs / hbm_peak, "traffic": committed_traffic(w.name),
                         "frac_isolated": frac_iso, "isolated_launch_us": iso_us,
                         "isolated_source": "profiles/ncu_bypass_summary.json (ncu gpu__time_duration, cold L2, "
                                            "one launch alone)",
                         "peak_kind": peak_kind, "kernel": " + ".join(kernel_names[p] for p in paths),
                         "scope": f"one step = {launches_per_step} launch(es); bytes and time of the whole step "
                                  f"(pipelined: consecutive independent steps overlap through PDL -- prologues, and "
                                  f"for the all-to-all kernel the X / Y loads once the launcher proved the preceding "
                                  f"step disjoint; see dependent_chain for strictly dependent steps)",
                         "step_us": kernel_us, "algorithmic_bytes_per_step": step_bytes},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_residual": e2e_res,
            "e2e_run_bypass": e2e_rb,
            "grouped": grouped,
            "layer_forward": layer_fwd,
            "clocks": clocks,
            "gpu_launches": int(args.steps * launches_per_step),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def impl_ours_merge(args):
    """cfg4: merge W(4096 x 11008, bf16) += down.up for all 32 layers per step."""
    import torch

    rank, world, local = dist_setup(args.gpus)
    import paper_2411_00915_b200 as atmm
    from paper_2411_00915_b200.workloads import MergeWorkload

    mw = MergeWorkload()
    dev = torch.device("cuda", local)
    reg = atmm.AdapterRegistry(mw.layers, mw.d_in, mw.d_out, device=local)
    rng = np.random.default_rng(5 + rank)
    s = 1.0 / np.sqrt(mw.rank)
    reg.put(1, rng.uniform(-s, s, (mw.layers, mw.d_in, mw.rank)).astype(np.float32),
            rng.uniform(-s, s, (mw.layers, mw.rank, mw.d_out)).astype(np.float32))
    W = torch.empty(mw.layers, mw.d_in, mw.d_out, dtype=torch.bfloat16, device=dev).uniform_(-0.02, 0.02)
    stream = torch.cuda.Stream(device=dev)

    def step(i):
        sign = 1.0 if i % 2 == 0 else -1.0  # merge, unmerge, merge, ... (all layers, one launch)
        atmm.merge_layers_into(reg, 1, W, sign=sign, stream=stream)

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
        for i in range(args.steps):
            step(i)
    g.replay()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    t_end = time.perf_counter() + args.soak_s
    while time.perf_counter() < t_end:
        g.replay()
        torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    per_step_ms = ms / args.steps
    hbm_peak, peak_kind = measured_peaks()
    bytes_step = mw.bytes(2)
    # ---- mode switch (serving.hpp:38-74): swap a new 32-layer adapter in from
    # pinned host memory (H2D + device-side packing, stream-ordered) and merge
    # it into every layer; device time, CUDA events ----
    dn = torch.from_numpy(rng.uniform(-s, s, (mw.layers, mw.d_in, mw.rank)).astype(np.float32)).pin_memory()
    upf = torch.from_numpy(rng.uniform(-s, s, (mw.layers, mw.rank, mw.d_out)).astype(np.float32)).pin_memory()
    sw = []
    for rep in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            reg.put_async(2, dn, upf, stream=stream)
            e1.record(stream)
            atmm.merge_layers_into(reg, 2, W, sign=1.0 if rep % 2 == 0 else -1.0, stream=stream)
            e2.record(stream)
        torch.cuda.synchronize()
        sw.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    swap_ms, merge_ms = min(sw, key=lambda v: v[0] + v[1])
    mode_switch = {"adapter_swap_ms": swap_ms, "merge_all_layers_ms": merge_ms, "total_ms": swap_ms + merge_ms,
                   "h2d_bytes": int(dn.numel() + upf.numel()) * 4,
                   "note": "put_async (pinned fp32 factors, 32 layers, r64) + one-launch merge of all layers"}
    achieved = bytes_step / (per_step_ms * 1e-3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = cpu_threads()
            el, rate = reference_merge_rate(mw, threads, 2)
            _, one = reference_merge_rate(mw, 1, 1)
            cpu = {"value": rate, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
                   "sample": f"2 cfg4 layers (4096 x 11008, r64, fp32) through the reference's delta_w_into + "
                             f"add_inplace, LORASERVE_THREADS={threads}: {el * 1e3:.0f} ms per layer",
                   "cpu_model": cpu_model(), "value_1thread": one}
        except FileNotFoundError as e:
            cpu = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps({
            "metric": "ATMM merge/unmerge W +- s.down.up, all 32 layers (mode switch) TFLOP/s", "value":
                world * mw.flops() / (per_step_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": merge_config(mw, world),
            "timing": {"l2": "W of 32 layers = 2.9 GB >> L2; K steps in one CUDA graph"},
            "cpu_baseline": cpu,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "atmm_merge_tma_kernel"},
            "mode_switch": mode_switch,
            "clocks": clocks, "gpu_launches": args.steps}), flush=True)


def main():
    args = parse_args()
    from paper_2411_00915_b200.workloads import bypass_config

    if args.config == "cfg4":
        if args.impl == "reference":
            impl_reference_merge(args)
            return
        impl_ours_merge(args)
        return
    w = bypass_config(args.config)
    if args.impl == "reference":
        impl_reference(args, w)
    else:
        impl_ours_bypass(args, w)


if __name__ == "__main__":
    main()
