"""B200-native ATMM (VaLoRA adaptive-tiling batched-LoRA operator).

Public API mirrors the reference loraserve operator interface; see
``paper_2411_00915_b200.atmm`` and include/atmm_b200.h.
"""
from .atmm import (  # noqa: F401
    BF16,
    F32,
    AdapterRegistry,
    BatchPlan,
    BypassPlan,
    ConfigError,
    CudaError,
    Error,
    IoError,
    MixturePlan,
    ModeError,
    NoDeviceError,
    ParseError,
    Segment,
    ShapeError,
    TilingConfig,
    TilingTable,
    UnknownAdapterError,
    atmm_multiply,
    bench_launches,
    candidate_configs,
    default_candidates,
    delta_w,
    device_count,
    heuristic_launch,
    m_bucket_of,
    merge_into,
    plan_batch,
    plan_batch_csr,
    residual_host_bf16_pipelined,
    run_bypass,
    shard_rows,
)
