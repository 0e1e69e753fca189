"""ctypes wrappers of the parity checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle``  -- oracle/_build/liboracle.so, the C restatement of the
  reference hot path (oracle/atmm_oracle.c).
* ``Reference`` -- oracle/_ref/libloraserve_ref.so, the UNMODIFIED reference
  headers compiled in place by oracle/Makefile (present wherever it was built;
  /root/reference itself is never read at run time).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_long, c_size_t, c_uint64, c_void_p

import numpy as np
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libloraserve_ref.so")

f32p = POINTER(c_float)
f64p = POINTER(c_double)
i32p = POINTER(c_int32)
i64p = POINTER(c_int64)
u64p = POINTER(c_uint64)


def _p(a, t):
    return a.ctypes.data_as(t)


def _ptr_array(arrs):
    return (c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = ctypes.CDLL(path)
        self.L = L
        L.orc_rng_size.restype = c_size_t
        L.orc_rng_next.restype = c_uint64
        L.orc_uniform.restype = c_float
        L.orc_uniform.argtypes = [c_void_p, c_float, c_float]
        L.orc_fill_uniform.argtypes = [c_void_p, f32p, c_size_t, c_float, c_float]
        L.orc_rng_seed.argtypes = [c_void_p, c_uint64]
        L.orc_rng_next.argtypes = [c_void_p]
        L.orc_seeded_shuffle_u64.argtypes = [c_void_p, u64p, c_size_t]
        L.orc_adapter_random.argtypes = [c_uint64, c_size_t, c_size_t, c_size_t, f32p, f32p]
        L.orc_model_random.argtypes = [c_uint64, c_size_t, c_size_t, f32p]
        L.orc_round_bf16.argtypes = [f32p, c_size_t]
        L.orc_gemm_reference.argtypes = [f32p, f32p, f32p, c_size_t, c_size_t, c_size_t]
        L.orc_gemm_reference_f64.argtypes = [f32p, f32p, f64p, c_size_t, c_size_t, c_size_t]
        L.orc_config_valid.argtypes = [i32p]
        L.orc_atmm_multiply.argtypes = [f32p, f32p, f32p, c_size_t, c_size_t, c_size_t, i32p]
        L.orc_add_inplace.argtypes = [f32p, f32p, c_size_t]
        L.orc_sub_inplace.argtypes = [f32p, f32p, c_size_t]
        L.orc_max_abs_diff.restype = c_double
        L.orc_max_abs_diff.argtypes = [f32p, f32p, c_size_t]
        L.orc_max_abs.restype = c_double
        L.orc_max_abs.argtypes = [f32p, c_size_t]
        L.orc_m_bucket_of.restype = c_int32
        L.orc_m_bucket_of.argtypes = [c_uint64]
        L.orc_table_lookup.argtypes = [i32p, i32p, c_size_t, i32p, c_uint64, c_uint64, c_uint64, i32p]
        L.orc_plan_batch.restype = c_long
        L.orc_plan_batch.argtypes = [i32p, c_size_t, i32p, i64p, i64p]
        L.orc_run_bypass.argtypes = [f32p, c_size_t, c_size_t, i32p, c_size_t, i32p, i64p, c_void_p, c_void_p, f32p]
        L.orc_bypass_rows_f64.argtypes = [f32p, c_size_t, c_size_t, c_size_t, i32p, c_size_t, i32p, i64p, c_void_p,
                                          c_void_p, f64p]
        L.orc_delta_w.argtypes = [f32p, f32p, c_size_t, c_size_t, c_size_t, f32p]
        L.orc_merge.argtypes = [f32p, c_size_t, c_size_t, c_size_t, c_size_t, f32p, f32p, c_int]
        L.orc_forward_f64.argtypes = [f32p, c_size_t, c_size_t, c_size_t, f32p, c_int, i32p, ctypes.c_int32, c_size_t,
                                      i32p, i64p, c_void_p, c_void_p, c_int, f64p]

    # ---- RNG ----
    def rng(self, seed: int):
        st = ctypes.create_string_buffer(self.L.orc_rng_size())
        self.L.orc_rng_seed(st, seed)
        return st

    def fill_uniform(self, rng, count: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        out = np.zeros(count, np.float32)
        self.L.orc_fill_uniform(rng, _p(out, f32p), count, lo, hi)
        return out

    def random_matrix(self, rng, rows: int, cols: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        return self.fill_uniform(rng, rows * cols, lo, hi).reshape(rows, cols)

    def seeded_shuffle(self, rng, v) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(v, np.uint64))
        self.L.orc_seeded_shuffle_u64(rng, _p(a, u64p), a.size)
        return a

    def adapter_random(self, seed: int, L: int, d: int, r: int):
        down = np.zeros((L, d, r), np.float32)
        up = np.zeros((L, r, d), np.float32)
        self.L.orc_adapter_random(seed, L, d, r, _p(down, f32p), _p(up, f32p))
        return down, up

    def model_random(self, seed: int, L: int, d: int) -> np.ndarray:
        w = np.zeros((L, d, d), np.float32)
        self.L.orc_model_random(seed, L, d, _p(w, f32p))
        return w

    @staticmethod
    def round_bf16(x: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(np.array(x, np.float32, copy=True))
        u = a.view(np.uint32)
        nan = ((u & 0x7F800000) == 0x7F800000) & ((u & 0x007FFFFF) != 0)
        r = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
        r = np.where(nan, (u | 0x00400000) & 0xFFFF0000, r).astype(np.uint32)
        return r.view(np.float32).reshape(a.shape)

    # ---- matrix core ----
    def gemm_reference(self, a, b) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.float32)
        self.L.orc_gemm_reference(_p(a, f32p), _p(b, f32p), _p(c, f32p), m, k, n)
        return c

    def gemm_reference_f64(self, a, b) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.float64)
        self.L.orc_gemm_reference_f64(_p(a, f32p), _p(b, f32p), _p(c, f64p), m, k, n)
        return c

    def config_valid(self, cfg) -> bool:
        return bool(self.L.orc_config_valid(_p(np.asarray(cfg, np.int32), i32p)))

    def atmm_multiply(self, a, b, cfg=(64, 32, 32, 32, 32, 32)) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.float32)
        st = self.L.orc_atmm_multiply(_p(a, f32p), _p(b, f32p), _p(c, f32p), m, k, n,
                                      _p(np.asarray(cfg, np.int32), i32p))
        if st != 0:
            raise ValueError(f"oracle status {st}")
        return c

    def m_bucket_of(self, m: int) -> int:
        return int(self.L.orc_m_bucket_of(m))

    def table_lookup(self, entries, default, m, k, n):
        """entries: list of ((m_bucket, k, n), cfg6)."""
        keys = np.asarray([e[0] for e in entries] or [[0, 0, 0]], np.int32).reshape(-1)
        cfgs = np.asarray([e[1] for e in entries] or [[0] * 6], np.int32).reshape(-1)
        out = np.zeros(6, np.int32)
        self.L.orc_table_lookup(_p(keys, i32p), _p(cfgs, i32p), len(entries), _p(np.asarray(default, np.int32), i32p),
                                m, k, n, _p(out, i32p))
        return tuple(int(v) for v in out)

    # ---- batch ----
    def plan_batch(self, assignment):
        a = np.ascontiguousarray(np.asarray(assignment, np.int32))
        n = a.size
        seg = np.zeros(max(n, 1), np.int32)
        off = np.zeros(max(n, 1) + 1, np.int64)
        rows = np.zeros(max(n, 1), np.int64)
        S = self.L.orc_plan_batch(_p(a, i32p), n, _p(seg, i32p), _p(off, i64p), _p(rows, i64p))
        if S < 0:
            raise ValueError("empty assignment")
        return seg[:S].copy(), off[: S + 1].copy(), rows[:n].copy()

    def run_bypass(self, x, assignment, adapters: dict) -> np.ndarray:
        """adapters: id -> (down d x r, up r x d) for one layer."""
        x = np.ascontiguousarray(x, np.float32)
        a = np.ascontiguousarray(np.asarray(assignment, np.int32))
        ids = np.asarray(sorted(adapters), np.int32)
        downs = [np.ascontiguousarray(adapters[i][0], np.float32) for i in ids]
        ups = [np.ascontiguousarray(adapters[i][1], np.float32) for i in ids]
        ranks = np.asarray([d.shape[1] for d in downs], np.int64)
        n, d = x.shape
        out = np.zeros((n, ups[0].shape[1] if ups else d), np.float32)
        st = self.L.orc_run_bypass(_p(x, f32p), n, d, _p(a, i32p), len(ids), _p(ids, i32p), _p(ranks, i64p),
                                   _ptr_array(downs), _ptr_array(ups), _p(out, f32p))
        if st != 0:
            raise KeyError(f"oracle status {st}")
        return out

    def bypass_rows_f64(self, x, assignment, adapters: dict) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        a = np.ascontiguousarray(np.asarray(assignment, np.int32))
        ids = np.asarray(sorted(adapters), np.int32)
        downs = [np.ascontiguousarray(adapters[i][0], np.float32) for i in ids]
        ups = [np.ascontiguousarray(adapters[i][1], np.float32) for i in ids]
        ranks = np.asarray([d.shape[1] for d in downs], np.int64)
        n, d_in = x.shape
        d_out = ups[0].shape[1]
        out = np.zeros((n, d_out), np.float64)
        st = self.L.orc_bypass_rows_f64(_p(x, f32p), n, d_in, d_out, _p(a, i32p), len(ids), _p(ids, i32p),
                                        _p(ranks, i64p), _ptr_array(downs), _ptr_array(ups), _p(out, f64p))
        if st != 0:
            raise KeyError(f"oracle status {st}")
        return out

    def forward_f64(self, x, w, mode: str = "unmerged", assignment=None, adapters: Optional[dict] = None,
                    merged_id: int = -1, round_act: bool = True) -> np.ndarray:
        """Stack forward (model.hpp:192-328), mode 'unmerged' | 'merged' |
        'mixture'.  w: [L][d][d]; adapters: {id: (down [L][d][r], up [L][r][d])};
        for 'mixture' w must already hold the merged adapter."""
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        n, d = x.shape
        L = w.shape[0]
        m = {"unmerged": 0, "merged": 1, "mixture": 2}[mode]
        adapters = adapters or {}
        ids = np.asarray(sorted(adapters), np.int32)
        downs = [np.ascontiguousarray(adapters[i][0], np.float32) for i in ids]
        ups = [np.ascontiguousarray(adapters[i][1], np.float32) for i in ids]
        ranks = np.asarray([dn.shape[-1] for dn in downs], np.int64)
        a = np.ascontiguousarray(np.asarray(assignment if assignment is not None else np.zeros(n), np.int32))
        out = np.zeros((n, d), np.float64)
        st = self.L.orc_forward_f64(_p(x, f32p), n, d, L, _p(w, f32p), m, _p(a, i32p), merged_id, len(ids),
                                    _p(ids, i32p), _p(ranks, i64p), _ptr_array(downs), _ptr_array(ups),
                                    1 if round_act else 0, _p(out, f64p))
        if st != 0:
            raise KeyError(f"oracle status {st}")
        return out

    def delta_w(self, down, up) -> np.ndarray:
        down = np.ascontiguousarray(down, np.float32)
        up = np.ascontiguousarray(up, np.float32)
        d_in, r = down.shape
        d_out = up.shape[1]
        out = np.zeros((d_in, d_out), np.float32)
        self.L.orc_delta_w(_p(down, f32p), _p(up, f32p), d_in, r, d_out, _p(out, f32p))
        return out

    def merge(self, w, down, up, sign: int = 1) -> np.ndarray:
        """w: [L, d_in, d_out] (copied), down [L, d_in, r], up [L, r, d_out]."""
        w = np.ascontiguousarray(np.array(w, np.float32, copy=True))
        down = np.ascontiguousarray(down, np.float32)
        up = np.ascontiguousarray(up, np.float32)
        L, d_in, d_out = w.shape
        r = down.shape[2]
        self.L.orc_merge(_p(w, f32p), L, d_in, r, d_out, _p(down, f32p), _p(up, f32p), sign)
        return w

    @staticmethod
    def max_abs_diff(a, b) -> float:
        return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)))) if np.size(a) else 0.0


class Reference:
    """The reference itself (compiled by oracle/Makefile into oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it where /root/reference is mounted (make -C oracle)")
        L = ctypes.CDLL(path)
        self.L = L
        L.ref_rng_new.restype = c_void_p
        L.ref_rng_new.argtypes = [c_uint64]
        L.ref_rng_free.argtypes = [c_void_p]
        L.ref_rng_next.restype = c_uint64
        L.ref_rng_next.argtypes = [c_void_p]
        L.ref_fill_uniform.argtypes = [c_void_p, f32p, c_size_t, c_float, c_float]
        L.ref_seeded_shuffle_u64.argtypes = [c_void_p, u64p, c_size_t]
        L.ref_adapter_random.argtypes = [c_int, c_size_t, c_size_t, c_size_t, c_uint64, f32p, f32p]
        L.ref_model_random.argtypes = [c_size_t, c_size_t, c_size_t, c_uint64, f32p]
        L.ref_gemm_reference.argtypes = [f32p, f32p, f32p, c_size_t, c_size_t, c_size_t]
        L.ref_atmm_multiply.argtypes = [f32p, c_size_t, c_size_t, f32p, c_size_t, c_size_t, f32p, i32p]
        L.ref_add_inplace.argtypes = [f32p, f32p, c_size_t]
        L.ref_sub_inplace.argtypes = [f32p, f32p, c_size_t]
        L.ref_m_bucket_of.argtypes = [c_uint64]
        L.ref_config_valid.argtypes = [i32p]
        L.ref_candidate_count.argtypes = [c_size_t, c_size_t]
        L.ref_candidate_configs.argtypes = [c_size_t, c_size_t, i32p, c_size_t]
        L.ref_default_candidates.argtypes = [c_size_t, c_size_t, i32p, c_size_t]
        L.ref_table_lookup.argtypes = [i32p, i32p, c_size_t, i32p, c_uint64, c_uint64, c_uint64, i32p]
        L.ref_table_load_lookup.argtypes = [ctypes.c_char_p, c_uint64, c_uint64, c_uint64, i32p]
        L.ref_table_save.argtypes = [i32p, i32p, i64p, c_size_t, i32p, ctypes.c_char_p]
        L.ref_save_matrix.argtypes = [ctypes.c_char_p, c_size_t, c_size_t, f32p]
        L.ref_save_fixture.argtypes = [ctypes.c_char_p, c_size_t, c_size_t, c_size_t, c_uint64, c_size_t, i32p, i64p,
                                       f32p]
        L.ref_plan_batch.restype = c_long
        L.ref_plan_batch.argtypes = [i32p, c_size_t, i32p, i64p, i64p]
        L.ref_ctx_new.restype = c_void_p
        L.ref_ctx_new.argtypes = [c_size_t, c_size_t, i32p, i64p, c_void_p, c_void_p]
        L.ref_ctx_free.argtypes = [c_void_p]
        L.ref_ctx_run_bypass.argtypes = [c_void_p, f32p, c_size_t, i32p, f32p]
        L.ref_ctx_bypass_residual.argtypes = [c_void_p, f32p, c_size_t, i32p, f32p, i64p]
        L.ref_merge_rect.argtypes = [f32p, c_size_t, c_size_t, c_size_t, f32p, f32p, c_int, f32p, i64p]
        L.ref_model_merge_cycle.argtypes = [f32p, c_size_t, c_size_t, c_size_t, f32p, f32p, c_int]
        L.ref_forward.argtypes = [c_int, c_size_t, c_size_t, f32p, c_size_t, i32p, i64p, c_void_p, c_void_p, f32p,
                                  c_size_t, i32p, ctypes.c_int32, f32p]

    def fill_uniform(self, seed: int, count: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        h = self.L.ref_rng_new(seed)
        out = np.zeros(count, np.float32)
        self.L.ref_fill_uniform(h, _p(out, f32p), count, lo, hi)
        self.L.ref_rng_free(h)
        return out

    def adapter_random(self, id_: int, L: int, d: int, r: int, seed: int):
        down = np.zeros((L, d, r), np.float32)
        up = np.zeros((L, r, d), np.float32)
        st = self.L.ref_adapter_random(id_, L, d, r, seed, _p(down, f32p), _p(up, f32p))
        if st != 0:
            raise ValueError(f"reference status {st}")
        return down, up

    def plan_batch(self, assignment):
        a = np.ascontiguousarray(np.asarray(assignment, np.int32))
        n = a.size
        seg = np.zeros(max(n, 1), np.int32)
        off = np.zeros(max(n, 1) + 1, np.int64)
        rows = np.zeros(max(n, 1), np.int64)
        S = self.L.ref_plan_batch(_p(a, i32p), n, _p(seg, i32p), _p(off, i64p), _p(rows, i64p))
        if S < 0:
            raise ValueError(f"reference status {-S}")
        return seg[:S].copy(), off[: S + 1].copy(), rows[:n].copy()

    def atmm_multiply(self, a, b, cfg) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        c = np.zeros((a.shape[0], b.shape[1]), np.float32)
        st = self.L.ref_atmm_multiply(_p(a, f32p), a.shape[0], a.shape[1], _p(b, f32p), b.shape[0], b.shape[1],
                                      _p(c, f32p), _p(np.asarray(cfg, np.int32), i32p))
        if st != 0:
            raise ValueError(f"reference status {st}")
        return c

    def gemm_reference(self, a, b) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        c = np.zeros((a.shape[0], b.shape[1]), np.float32)
        self.L.ref_gemm_reference(_p(a, f32p), _p(b, f32p), _p(c, f32p), a.shape[0], a.shape[1], b.shape[1])
        return c

    class Ctx:
        def __init__(self, ref, d: int, adapters: dict):
            self.ref = ref
            ids = np.asarray(sorted(adapters), np.int32)
            self.downs = [np.ascontiguousarray(adapters[i][0], np.float32) for i in ids]
            self.ups = [np.ascontiguousarray(adapters[i][1], np.float32) for i in ids]
            ranks = np.asarray([x.shape[1] for x in self.downs], np.int64)
            self.d = d
            self.h = ref.L.ref_ctx_new(d, len(ids), _p(ids, i32p), _p(ranks, i64p), _ptr_array(self.downs),
                                       _ptr_array(self.ups))
            if not self.h:
                raise ValueError("reference rejected the adapters")

        def run_bypass(self, x, assignment) -> np.ndarray:
            x = np.ascontiguousarray(x, np.float32)
            a = np.ascontiguousarray(np.asarray(assignment, np.int32))
            out = np.zeros((x.shape[0], self.d), np.float32)
            st = self.ref.L.ref_ctx_run_bypass(self.h, _p(x, f32p), x.shape[0], _p(a, i32p), _p(out, f32p))
            if st != 0:
                raise KeyError(f"reference status {st}")
            return out

        def bypass_residual(self, x, assignment, y) -> int:
            """y += run_bypass(x) in place; returns elapsed ns (reference's own clock)."""
            el = c_int64(0)
            st = self.ref.L.ref_ctx_bypass_residual(self.h, _p(x, f32p), x.shape[0], _p(assignment, i32p),
                                                    _p(y, f32p), ctypes.byref(el))
            if st != 0:
                raise KeyError(f"reference status {st}")
            return el.value

        def __del__(self):
            if getattr(self, "h", None):
                self.ref.L.ref_ctx_free(self.h)
                self.h = None

    def ctx(self, d: int, adapters: dict) -> "Reference.Ctx":
        return Reference.Ctx(self, d, adapters)

    def forward(self, x, w, mode: str = "unmerged", assignment=None, adapters: Optional[dict] = None,
                merged_id: int = -1):
        """The reference's forward_unmerged / forward_merged / forward_mixture.
        Returns (out fp32, weights after the call: merged for 'mixture')."""
        x = np.ascontiguousarray(x, np.float32)
        w = np.array(w, np.float32, copy=True, order="C")
        n, d = x.shape
        L = w.shape[0]
        m = {"unmerged": 0, "merged": 1, "mixture": 2}[mode]
        adapters = adapters or {}
        ids = np.asarray(sorted(adapters), np.int32)
        downs = [np.ascontiguousarray(adapters[i][0], np.float32) for i in ids]
        ups = [np.ascontiguousarray(adapters[i][1], np.float32) for i in ids]
        ranks = np.asarray([dn.shape[-1] for dn in downs], np.int64)
        a = np.ascontiguousarray(np.asarray(assignment if assignment is not None else np.zeros(n), np.int32))
        out = np.zeros((n, d), np.float32)
        st = self.L.ref_forward(m, L, d, _p(w, f32p), len(ids), _p(ids, i32p), _p(ranks, i64p), _ptr_array(downs),
                                _ptr_array(ups), _p(x, f32p), n, _p(a, i32p), merged_id, _p(out, f32p))
        if st != 0:
            raise ValueError(f"reference status {st}")
        return out, w

    def merge_rect(self, w, down, up, sign: int = 1):
        """In place on w (d_in x d_out fp32); returns elapsed ns."""
        d_in, r = down.shape
        d_out = up.shape[1]
        scratch = np.zeros((d_in, d_out), np.float32)
        el = c_int64(0)
        st = self.L.ref_merge_rect(_p(w, f32p), d_in, r, d_out, _p(np.ascontiguousarray(down), f32p),
                                   _p(np.ascontiguousarray(up), f32p), sign, _p(scratch, f32p), ctypes.byref(el))
        if st != 0:
            raise ValueError(f"reference status {st}")
        return el.value
