"""B200-native ATMM (VaLoRA adaptive-tiling batched-LoRA operator).

Public API mirrors the reference loraserve operator interface; see
``paper_2411_00915_b200.atmm`` and include/atmm_b200.h.

The operator names are resolved lazily: ``import paper_2411_00915_b200`` and
its pure-Python submodules (``workloads``) do not load libatmm_b200.so; the
first access to an operator name imports ``.atmm``, which loads the library
and fails loudly if it is missing (there is no CPU fallback).
"""
from __future__ import annotations

import importlib

_ATMM_NAMES = (
    "BF16", "F32", "AdapterRegistry", "BatchPlan", "BypassPlan", "ConfigError", "CudaError", "Error", "IoError",
    "LayerForward", "MixturePlan", "ModeError", "ModelState", "NoDeviceError", "ParseError", "Segment", "ShapeError",
    "TilingConfig", "TilingTable", "UnknownAdapterError", "atmm_multiply", "candidate_configs",
    "default_candidates", "delta_w", "device_count", "fixture_info", "forward_merged", "forward_mixture",
    "forward_unmerged", "gemm", "load_matrix", "heuristic_launch", "m_bucket_of", "merge_into", "merge_layers_into",
    "plan_batch", "plan_batch_csr", "residual_host_bf16_pipelined", "run_bypass", "run_bypass_host_bf16_pipelined",
    "save_matrix", "shard_rows", "flops_read", "flops_reset", "FlopScope", "bypass_flops",
    "TuneShape", "default_shape_grid", "default_launch_candidates", "benchmark_launch", "grid_bench_ns",
    "tiling_search", "table_from_scores", "gemm_f32", "forward_f32", "UNMERGED", "MERGED", "MIXTURE",
    "default_table", "DEFAULT_TABLE_PATH", "overlap_stats", "split_overlap_stats",
)

__all__ = list(_ATMM_NAMES)


def __getattr__(name):
    if name in _ATMM_NAMES:
        mod = importlib.import_module(".atmm", __name__)
        val = getattr(mod, name)
        globals()[name] = val
        return val
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
