"""ctypes binding of libatmm_b200.so (include/atmm_b200.h).

The shared library is built in-tree by ``paper_2411_00915_b200.build`` (or
``python -c "import __graft_entry__ as g; g.build()"``).  There is no fallback:
if the library is missing, importing this module fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t, c_uint16, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libatmm_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2411_00915_b200.build` "
        "(the ATMM operator has no CPU / PyTorch fallback)"
    )

lib = ctypes.CDLL(LIB_PATH)

i32p = POINTER(c_int32)
i64p = POINTER(c_int64)
f32p = POINTER(c_float)
u16p = POINTER(c_uint16)

_SIGS = {
    "atmm_last_error": (c_char_p, []),
    "atmm_abi_version": (c_int, []),
    "atmm_device_count": (c_int, []),
    "atmm_overlap_stats": (c_int, [i64p, i64p]),
    "atmm_split_overlap_stats": (c_int, [i64p, i64p]),
    "atmm_flops_read": (ctypes.c_uint64, []),
    "atmm_flops_reset": (None, []),
    "atmm_bypass_flops": (c_int, [i32p, c_int64, i32p, i64p, c_int64, c_int64, c_int64, POINTER(ctypes.c_uint64)]),
    "atmm_state_create": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, POINTER(c_void_p)]),
    "atmm_state_destroy": (None, [c_void_p]),
    "atmm_state_get": (c_int, [c_void_p, POINTER(c_int), i32p, i64p]),
    "atmm_state_merge": (c_int, [c_void_p, c_int32, c_void_p]),
    "atmm_state_unmerge": (c_int, [c_void_p, c_int32, c_void_p]),
    "atmm_state_set_mixture": (c_int, [c_void_p, c_int32]),
    "atmm_state_mode_switch": (c_int, [c_void_p, c_int, c_int32, c_void_p, i64p]),
    "atmm_registry_set_precise": (c_int, [c_void_p, c_int]),
    "atmm_gemm_f32": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64,
                              c_float, c_void_p]),
    "atmm_bypass_apply_f32": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_float, c_void_p]),
    "atmm_merge_apply_f32": (c_int, [c_void_p, c_int32, c_int64, c_int64, c_void_p, c_int64, c_int64, c_float,
                                     c_void_p]),
    "atmm_delta_w_f32": (c_int, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_void_p]),
    "atmm_forward_f32": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                 c_int64, POINTER(c_void_p), f32p, c_int64, c_void_p]),
    "atmm_forward_f32_host": (c_int, [f32p, c_int64, c_int64, c_int64, f32p, f32p, POINTER(c_void_p), f32p, c_int64]),
    "atmm_merge_f32_host": (c_int, [c_void_p, c_int32, f32p, c_float]),
    "atmm_plan_batch": (c_int, [i32p, c_int64, i32p, i64p, i64p, i64p]),
    "atmm_config_valid": (c_int, [i32p]),
    "atmm_m_bucket_of": (c_int, [c_int64]),
    "atmm_table_create": (c_int, [i32p, POINTER(c_void_p)]),
    "atmm_table_destroy": (None, [c_void_p]),
    "atmm_table_insert": (c_int, [c_void_p, c_int32, c_int32, c_int32, i32p, c_int64, i32p]),
    "atmm_table_set_default": (c_int, [c_void_p, i32p, i32p]),
    "atmm_table_lookup": (c_int, [c_void_p, c_int64, c_int64, c_int64, i32p]),
    "atmm_table_size": (c_int, [c_void_p, i64p]),
    "atmm_table_find": (c_int, [c_void_p, c_int64, c_int64, c_int64, i32p, POINTER(c_int)]),
    "atmm_table_resolve_launch": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64, i32p]),
    "atmm_table_save": (c_int, [c_void_p, c_char_p]),
    "atmm_table_load": (c_int, [c_char_p, POINTER(c_void_p)]),
    "atmm_candidate_configs": (c_int, [c_size_t, c_size_t, i32p, c_size_t, POINTER(c_size_t)]),
    "atmm_default_candidates": (c_int, [c_size_t, c_size_t, i32p, c_size_t, POINTER(c_size_t)]),
    "atmm_registry_create": (c_int, [c_int, c_int64, c_int64, c_int64, POINTER(c_void_p)]),
    "atmm_registry_destroy": (None, [c_void_p]),
    "atmm_registry_put": (c_int, [c_void_p, c_int32, c_int64, f32p, f32p, c_float]),
    "atmm_registry_remove": (c_int, [c_void_p, c_int32]),
    "atmm_registry_contains": (c_int, [c_void_p, c_int32]),
    "atmm_registry_rank": (c_int, [c_void_p, c_int32, i64p]),
    "atmm_registry_bytes": (c_int, [c_void_p, i64p]),
    "atmm_plan_create": (c_int, [c_void_p, i32p, c_int64, c_void_p, POINTER(c_void_p)]),
    "atmm_plan_create_mapped": (c_int, [c_void_p, i32p, i32p, c_int64, c_int64, c_void_p, POINTER(c_void_p)]),
    "atmm_registry_put_combined": (c_int, [c_void_p, c_int32, c_int64, i32p, f32p]),
    "atmm_registry_put_async": (c_int, [c_void_p, c_int32, c_int64, f32p, f32p, c_float, c_void_p]),
    "atmm_registry_load_fixture": (c_int, [c_void_p, c_char_p, i64p]),
    "atmm_matrix_save": (c_int, [c_char_p, c_int64, c_int64, f32p]),
    "atmm_matrix_load": (c_int, [c_char_p, i64p, i64p, f32p, c_int64]),
    "atmm_fixture_info": (c_int, [c_char_p, i64p, i64p, i64p, i32p, i64p, c_int64]),
    "atmm_run_bypass_host_bf16_pipelined": (c_int, [c_void_p, i64p, POINTER(c_void_p), POINTER(c_void_p), c_int64]),
    "atmm_bypass_apply_group": (c_int, [c_void_p, c_int64, i64p, POINTER(c_void_p), c_int64, POINTER(c_void_p),
                                        c_int64, c_int, c_float, c_void_p]),
    "atmm_merge_apply_layers": (c_int, [c_void_p, c_int32, c_int64, c_int64, c_void_p, c_int64, c_int64, c_int,
                                        c_float, c_void_p]),
    "atmm_plan_destroy": (None, [c_void_p]),
    "atmm_plan_set_flags": (c_int, [c_void_p, ctypes.c_uint32]),
    "atmm_forward_create": (c_int, [c_void_p, c_int, c_int64, c_int64, POINTER(c_void_p)]),
    "atmm_forward_create_opts": (c_int, [c_void_p, c_int, c_int64, c_int64, c_void_p, POINTER(c_void_p)]),
    "atmm_gemm_ex": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int, c_int64, c_int64, c_int64,
                             c_void_p, c_void_p]),
    "atmm_forward_destroy": (None, [c_void_p]),
    "atmm_forward_run": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                 c_void_p]),
    "atmm_forward_stats": (c_int, [c_void_p, i64p, c_int64]),
    "atmm_gemm": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int, c_int64, c_int64, c_int64,
                          c_void_p]),
    "atmm_plan_routing": (c_int, [c_void_p, i32p, i64p, i64p, i64p]),
    "atmm_plan_stats": (c_int, [c_void_p, i64p, i64p, i64p]),
    "atmm_plan_describe": (c_int, [c_void_p, ctypes.c_char_p, c_size_t]),
    "atmm_bypass_apply": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int, c_float, c_void_p]),
    "atmm_run_bypass_host": (c_int, [c_void_p, f32p, c_int64, i32p, c_int64, c_void_p, f32p]),
    "atmm_bypass_residual_host_bf16": (c_int, [c_void_p, c_int64, u16p, u16p, c_float, c_void_p]),
    "atmm_bypass_residual_host_bf16_pipelined": (c_int, [c_void_p, i64p, POINTER(c_void_p), POINTER(c_void_p), c_int64, c_float]),
    "atmm_merge_apply": (c_int, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int, c_float, c_void_p]),
    "atmm_delta_w_host": (c_int, [c_void_p, c_int32, c_int64, f32p]),
    "atmm_multiply_host": (c_int, [f32p, c_int64, c_int64, f32p, c_int64, f32p, i32p]),
    "atmm_benchmark_launch": (c_int, [c_int, c_void_p, i32p, c_int, ctypes.c_uint64, i64p]),
    "atmm_grid_bench_ns": (c_int, [c_int, c_void_p, c_int64, i32p, c_int64, c_int, c_int, i64p, c_char_p, c_size_t]),
    "atmm_tiling_search": (c_int, [c_int, c_void_p, c_int64, i32p, c_int64, c_int, POINTER(c_void_p), c_char_p,
                                   c_size_t]),
    "atmm_default_shape_grid": (c_int, [c_int64, c_int64, i64p, c_int64, c_void_p, c_int64, i64p]),
    "atmm_default_launch_candidates": (c_int, [i32p, c_int64, i64p]),
    "atmm_table_from_scores": (c_int, [c_void_p, c_int64, i32p, c_int64, i64p, POINTER(c_void_p), c_char_p, c_size_t]),
    "atmm_plan_create_launch": (c_int, [c_void_p, i32p, c_int64, i32p, POINTER(c_void_p)]),
    "atmm_shard_rows": (c_int, [i32p, c_int64, i32p, i64p, c_int64, c_int64, c_int64, c_int32, i32p]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


def last_error() -> str:
    msg = lib.atmm_last_error()
    return msg.decode() if msg else ""
