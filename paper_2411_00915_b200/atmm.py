"""Python mirror of the reference's ATMM operator interface over the C ABI.

Names, argument meaning and error behaviour follow loraserve
(/root/reference/proj/include/loraserve): ``plan_batch`` (batch.hpp:28),
``run_bypass`` (batch.hpp:48), ``TilingConfig``/``TilingTable``
(tiling.hpp:22-254), ``delta_w``/``merge``/``unmerge`` (model.hpp:120-188),
``atmm_multiply`` (atmm.hpp:144).  Exceptions mirror errors.hpp.

Device work goes through libatmm_b200.so (hand-written sm_100a kernels);
torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from ._lib import f32p, i32p, i64p, last_error, lib, u16p

# --------------------------------------------------------------- errors ---


class Error(RuntimeError):
    """loraserve::Error (errors.hpp:10)."""

    code = 9


class ShapeError(Error):
    code = 1


class ConfigError(Error):
    code = 2


class ModeError(Error):
    code = 3


class IoError(Error):
    code = 4


class ParseError(Error):
    code = 5


class UnknownAdapterError(Error):
    code = 6


class CudaError(Error):
    code = 7


class NoDeviceError(Error):
    code = 8


_BY_CODE = {c.code: c for c in (ShapeError, ConfigError, ModeError, IoError, ParseError,
                                 UnknownAdapterError, CudaError, NoDeviceError)}

BF16 = 0
F32 = 1


def _check(status: int) -> None:
    if status != 0:
        raise _BY_CODE.get(status, Error)(last_error())


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def device_count() -> int:
    """Number of visible sm_100 devices (0 on a CPU host)."""
    return int(lib.atmm_device_count())


# ---------------------------------------------------------------- flops ---


def flops_read() -> int:
    """flops.hpp:15: this thread's algorithmic FLOP counter."""
    return int(lib.atmm_flops_read())


def flops_reset() -> None:
    lib.atmm_flops_reset()


class FlopScope:
    """flops::Scope (flops.hpp:18-24): FLOPs counted since construction."""

    def __init__(self):
        self.start = flops_read()

    def elapsed(self) -> int:
        return flops_read() - self.start


def bypass_flops(assignment: Sequence[int], adapter_ranks: dict, d_in: int, d_out: Optional[int] = None) -> int:
    """Algorithmic FLOPs of one bypass pass (batch.hpp:45-47 via atmm.hpp:123):
    sum over plan_batch segments of 2 ns r (d_in + d_out).  Host only."""
    a = _i32(assignment).reshape(-1)
    ids = _i32(sorted(adapter_ranks))
    ranks = np.ascontiguousarray(np.asarray([adapter_ranks[i] for i in sorted(adapter_ranks)], np.int64))
    out = ctypes.c_uint64(0)
    _check(lib.atmm_bypass_flops(_p(a, i32p), a.size, _p(ids, i32p), _p(ranks, i64p), ids.size, int(d_in),
                                 int(d_in if d_out is None else d_out), ctypes.byref(out)))
    return int(out.value)


# -------------------------------------------------------------- planner ---


@dataclass
class Segment:
    adapter_id: int
    rows: List[int]


@dataclass
class BatchPlan:
    segments: List[Segment] = field(default_factory=list)
    total_rows: int = 0


def plan_batch_csr(assignment: Sequence[int]) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    a = _i32(assignment).reshape(-1)
    n = a.size
    seg = np.zeros(max(n, 1), np.int32)
    off = np.zeros(max(n, 1) + 1, np.int64)
    rows = np.zeros(max(n, 1), np.int64)
    S = ctypes.c_int64(0)
    _check(lib.atmm_plan_batch(_p(a, i32p), n, _p(seg, i32p), _p(off, i64p), _p(rows, i64p), ctypes.byref(S)))
    s = S.value
    return seg[:s].copy(), off[: s + 1].copy(), rows[:n].copy()


def plan_batch(assignment: Sequence[int]) -> BatchPlan:
    """batch.hpp:28-42: stable group-by, segments in ascending adapter id."""
    seg, off, rows = plan_batch_csr(assignment)
    plan = BatchPlan(total_rows=int(len(rows)))
    for s in range(len(seg)):
        plan.segments.append(Segment(int(seg[s]), [int(r) for r in rows[off[s]:off[s + 1]]]))
    return plan


# --------------------------------------------------------------- tiling ---


class TilingConfig(tuple):
    """(outer_m, outer_n, outer_k, inner_m, inner_n, inner_k), tiling.hpp:22."""

    def __new__(cls, *edges):
        if len(edges) == 1 and not isinstance(edges[0], int):
            edges = tuple(edges[0])
        if len(edges) != 6:
            raise ConfigError("tiling config must have 6 edges")
        return super().__new__(cls, (int(e) for e in edges))

    def structurally_valid(self) -> bool:
        return bool(lib.atmm_config_valid(_p(_i32(self), i32p)))

    def validate(self) -> None:
        if not self.structurally_valid():
            raise ConfigError(f"invalid tiling config {tuple(self)}")

    def footprint_elems(self) -> int:
        om, on, ok = self[0], self[1], self[2]
        return om * ok + ok * on + om * on


def m_bucket_of(m: int) -> int:
    return int(lib.atmm_m_bucket_of(int(m)))


def candidate_configs(cache_budget_bytes: int, scalar_width: int) -> List[TilingConfig]:
    return _configs(lib.atmm_candidate_configs, cache_budget_bytes, scalar_width)


def default_candidates(cache_budget_bytes: int, scalar_width: int) -> List[TilingConfig]:
    return _configs(lib.atmm_default_candidates, cache_budget_bytes, scalar_width)


def _configs(fn, budget, width) -> List[TilingConfig]:
    count = ctypes.c_size_t(0)
    _check(fn(budget, width, None, 0, ctypes.byref(count)))
    out = np.zeros(6 * max(count.value, 1), np.int32)
    _check(fn(budget, width, _p(out, i32p), count.value, ctypes.byref(count)))
    return [TilingConfig(out[6 * i: 6 * i + 6]) for i in range(count.value)]


class TilingTable:
    """tiling.hpp:153-254 plus the B200 launch resolution."""

    def __init__(self, default: Optional[Sequence[int]] = None, _handle=None):
        if _handle is not None:
            self._h = _handle
            return
        h = ctypes.c_void_p()
        d = _i32(default) if default is not None else None
        _check(lib.atmm_table_create(_p(d, i32p) if d is not None else None, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # (module globals are None at interpreter exit)
            lib.atmm_table_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def insert(self, m_bucket: int, k: int, n: int, config: Sequence[int], measured_ns: int = 0,
               sm100: Optional[Sequence[int]] = None) -> None:
        """sm100: {tile_m, cluster, bn, stages[, path]} (path 0 = automatic)."""
        s = _launch5(sm100) if sm100 is not None else None
        _check(lib.atmm_table_insert(self._h, m_bucket, k, n, _p(_i32(config), i32p), int(measured_ns),
                                     _p(s, i32p) if s is not None else None))

    def set_default(self, config: Sequence[int], sm100: Optional[Sequence[int]] = None) -> None:
        s = _launch5(sm100) if sm100 is not None else None
        _check(lib.atmm_table_set_default(self._h, _p(_i32(config), i32p), _p(s, i32p) if s is not None else None))

    def lookup(self, m: int, k: int, n: int) -> TilingConfig:
        out = np.zeros(6, np.int32)
        _check(lib.atmm_table_lookup(self._h, m, k, n, _p(out, i32p)))
        return TilingConfig(out)

    def resolve_launch(self, m: int, d_in: int, rank: int, d_out: int) -> Tuple[int, int, int, int, int]:
        """{tile_m, cluster, bn, stages, path} for a segment of m rows."""
        out = np.zeros(5, np.int32)
        _check(lib.atmm_table_resolve_launch(self._h, m, d_in, rank, d_out, _p(out, i32p)))
        return tuple(int(v) for v in out)

    def __len__(self) -> int:
        s = ctypes.c_int64(0)
        _check(lib.atmm_table_size(self._h, ctypes.byref(s)))
        return s.value

    def find_entry(self, m: int, k: int, n: int) -> Optional[Tuple[int, ...]]:
        """The B200 launch of the entry lookup(m, k, n) resolves to (exact or
        nearest bucket within 32, tiling.hpp:181-199), None on a miss."""
        out = np.zeros(5, np.int32)
        found = ctypes.c_int(0)
        _check(lib.atmm_table_find(self._h, m, k, n, _p(out, i32p), ctypes.byref(found)))
        return tuple(int(v) for v in out) if found.value else None

    def save(self, path: str) -> None:
        _check(lib.atmm_table_save(self._h, str(path).encode()))

    @classmethod
    def load(cls, path: str) -> "TilingTable":
        h = ctypes.c_void_p()
        _check(lib.atmm_table_load(str(path).encode(), ctypes.byref(h)))
        return cls(_handle=h)


def _launch5(launch: Sequence[int]) -> np.ndarray:
    v = [int(x) for x in launch]
    if len(v) == 4:
        v.append(0)
    if len(v) != 5:
        raise ConfigError("a launch is {tile_m, cluster, bn, stages[, path]}")
    return _i32(v)


def heuristic_launch(m: int, d_in: int, rank: int, d_out: int) -> Tuple[int, int, int, int, int]:
    out = np.zeros(5, np.int32)
    _check(lib.atmm_table_resolve_launch(None, m, d_in, rank, d_out, _p(out, i32p)))
    return tuple(int(v) for v in out)


# ------------------------------------------------------------- registry ---


class AdapterRegistry:
    """Device-resident AdapterSet (adapter.hpp:18-110) for one projection."""

    def __init__(self, num_layers: int, d_in: int, d_out: Optional[int] = None, device: int = 0,
                 precise: bool = False):
        """precise: also keep the fp32-faithful split images of every factor
        (atmm_registry_set_precise) for the fp32 entry points."""
        d_out = d_in if d_out is None else d_out
        h = ctypes.c_void_p()
        _check(lib.atmm_registry_create(device, num_layers, d_in, d_out, ctypes.byref(h)))
        self._h = h
        self.precise = bool(precise)
        if precise:
            _check(lib.atmm_registry_set_precise(h, 1))
        self.device = device
        self.num_layers, self.d_in, self.d_out = num_layers, d_in, d_out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # (module globals are None at interpreter exit)
            lib.atmm_registry_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def put(self, adapter_id: int, down, up, scale: float = 1.0) -> None:
        """down: [L, d_in, r] (or [d_in, r] for L = 1); up: [L, r, d_out]."""
        d = _f32(down)
        u = _f32(up)
        if d.ndim == 2:
            d = d[None]
        if u.ndim == 2:
            u = u[None]
        L, di, r = d.shape
        if L != self.num_layers or di != self.d_in or u.shape != (L, r, self.d_out):
            raise ShapeError(f"adapter factor shapes {d.shape} / {u.shape} do not match registry "
                             f"(L={self.num_layers}, d_in={self.d_in}, d_out={self.d_out})")
        _check(lib.atmm_registry_put(self._h, adapter_id, r, _p(d, f32p), _p(u, f32p), float(scale)))
        self._drop_combined(adapter_id)

    def _drop_combined(self, adapter_id: int) -> None:
        """Combined (mixture) slots built from adapter_id are stale now."""
        combos = self.__dict__.get("_combined", {})
        for key in [k for k in combos if adapter_id in k]:
            lib.atmm_registry_remove(self._h, combos.pop(key))

    def put_async(self, adapter_id: int, down, up, scale: float = 1.0, stream=None) -> None:
        """Adapter swap ordered on `stream` (H2D + device-side packing,
        atmm_registry_put_async).  down / up: numpy arrays or CPU torch tensors
        (pinned for an asynchronous copy; keep them alive until the stream
        has passed the copy)."""
        def host(a):
            try:
                import torch

                if isinstance(a, torch.Tensor):
                    t = a.detach().to(torch.float32).contiguous()
                    return t, ctypes.cast(t.data_ptr(), f32p), tuple(t.shape)
            except ImportError:
                pass
            arr = _f32(a)
            return arr, _p(arr, f32p), arr.shape

        dkeep, dptr, dshape = host(down)
        ukeep, uptr, ushape = host(up)
        if len(dshape) == 2:
            dshape = (1,) + tuple(dshape)
        if len(ushape) == 2:
            ushape = (1,) + tuple(ushape)
        L, di, r = dshape
        if L != self.num_layers or di != self.d_in or tuple(ushape) != (L, r, self.d_out):
            raise ShapeError(f"adapter factor shapes {dshape} / {ushape} do not match registry")
        sp = _stream_ptr(stream)
        _check(lib.atmm_registry_put_async(self._h, adapter_id, r, dptr, uptr, float(scale), sp))
        self._drop_combined(adapter_id)
        # The host factors must outlive the stream-ordered H2D copy: keep them
        # until an event recorded after the swap has completed, and drop every
        # kept pair whose swap is done (bounded: nothing outlives its copy).
        import torch

        ev = torch.cuda.Event()
        ev.record(torch.cuda.ExternalStream(sp, device=torch.device("cuda", self.device)))
        keep = [k for k in self.__dict__.get("_async_keep", []) if not k[0].query()]
        keep.append((ev, dkeep, ukeep))
        self._async_keep = keep

    def pending_swaps(self) -> int:
        """put_async swaps whose host buffers are still held (copy not yet done)."""
        return sum(1 for k in self.__dict__.get("_async_keep", []) if not k[0].query())

    def load_fixture(self, directory: str) -> int:
        """Every adapter of a reference fixture directory (manifest.json +
        binary matrices, model_io.hpp) into the registry; returns the count."""
        n = ctypes.c_int64(0)
        _check(lib.atmm_registry_load_fixture(self._h, str(directory).encode(), ctypes.byref(n)))
        return n.value

    def put_combined(self, new_id: int, parts: Sequence[Tuple[int, float]]) -> None:
        """A slot = rank-concatenation of existing adapters with signs folded
        into up (include/atmm_b200.h atmm_registry_put_combined): one fused
        bypass then adds sum_i sign_i s_i (x.down_i).up_i."""
        ids = _i32([p[0] for p in parts])
        signs = _f32([p[1] for p in parts])
        _check(lib.atmm_registry_put_combined(self._h, int(new_id), ids.size, _p(ids, i32p), _p(signs, f32p)))

    def remove(self, adapter_id: int) -> None:
        _check(lib.atmm_registry_remove(self._h, adapter_id))
        self._drop_combined(adapter_id)

    def __contains__(self, adapter_id: int) -> bool:
        return bool(lib.atmm_registry_contains(self._h, adapter_id))

    def rank(self, adapter_id: int) -> int:
        r = ctypes.c_int64(0)
        _check(lib.atmm_registry_rank(self._h, adapter_id, ctypes.byref(r)))
        return r.value

    def nbytes(self) -> int:
        b = ctypes.c_int64(0)
        _check(lib.atmm_registry_bytes(self._h, ctypes.byref(b)))
        return b.value


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def overlap_stats() -> Tuple[int, int]:
    """(all-to-all bypass launches, launches that started early) so far."""
    a, e = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib.atmm_overlap_stats(ctypes.byref(a), ctypes.byref(e)))
    return int(a.value), int(e.value)


def split_overlap_stats() -> Tuple[int, int]:
    """(split-path shrink + expand pairs launched, shrinks that started early) so far."""
    a, e = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib.atmm_split_overlap_stats(ctypes.byref(a), ctypes.byref(e)))
    return int(a.value), int(e.value)


class BypassPlan:
    """plan_batch + launch grouping for one batch on one registry."""

    def __init__(self, registry: AdapterRegistry, assignment: Sequence[int], table: Optional[TilingTable] = None,
                 rows: Optional[Sequence[int]] = None, n_rows: Optional[int] = None,
                 launch: Optional[Sequence[int]] = None, use_default_table: bool = True):
        """rows (optional): routed entry i is row rows[i] of X / Y, which
        have n_rows rows (atmm_plan_create_mapped); default: entry i = row i.
        launch (optional): {tile_m, cluster, bn, stages[, path]} forced for
        every segment instead of the table's (atmm_plan_create_launch).
        table None: the packaged B200-profiled table (default_table(); the
        built-in heuristic for shapes it does not cover), unless
        use_default_table is False (heuristic only)."""
        if table is None and launch is None and use_default_table:
            table = default_table()
        a = _i32(assignment).reshape(-1)
        h = ctypes.c_void_p()
        if launch is not None:
            if rows is not None:
                raise ConfigError("a forced launch takes no row map")
            _check(lib.atmm_plan_create_launch(registry.handle, _p(a, i32p), a.size, _p(_launch5(launch), i32p),
                                               ctypes.byref(h)))
            self.n = int(a.size)
        elif rows is None:
            _check(lib.atmm_plan_create(registry.handle, _p(a, i32p), a.size, table.handle if table else None,
                                        ctypes.byref(h)))
            self.n = int(a.size)
        else:
            rw = _i32(rows).reshape(-1)
            if rw.size != a.size or n_rows is None:
                raise ShapeError("rows must match the assignment length and n_rows must be given")
            _check(lib.atmm_plan_create_mapped(registry.handle, _p(a, i32p), _p(rw, i32p), a.size, int(n_rows),
                                               table.handle if table else None, ctypes.byref(h)))
            self.n = int(n_rows)
        self._h = h
        self.registry = registry
        self.n_routed = int(a.size)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # (module globals are None at interpreter exit)
            lib.atmm_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def set_x_ready(self, ready: bool = True) -> None:
        """ATMM_PLAN_X_READY: promise that the X of every apply is complete
        before the launch preceding the apply on its stream starts (e.g. the
        bypass follows the base GEMM Y = X W); X is then gathered under that
        launch's tail.  Results are unchanged."""
        self._flags = (getattr(self, "_flags", 0) & ~1) | (1 if ready else 0)
        _check(lib.atmm_plan_set_flags(self._h, self._flags))

    def set_overlap(self, allowed: bool = True) -> None:
        """ATMM_PLAN_NO_OVERLAP when not allowed: never start an apply's X / Y
        loads under the preceding launch (include/atmm_b200.h).  By default the
        launcher does so only when it proves the preceding launch touches
        disjoint bytes."""
        self._flags = (getattr(self, "_flags", 0) & ~2) | (0 if allowed else 2)
        _check(lib.atmm_plan_set_flags(self._h, self._flags))

    def routing(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        seg = np.zeros(self.n_routed, np.int32)
        off = np.zeros(self.n_routed + 1, np.int64)
        rows = np.zeros(self.n_routed, np.int64)
        S = ctypes.c_int64(0)
        _check(lib.atmm_plan_routing(self._h, _p(seg, i32p), _p(off, i64p), _p(rows, i64p), ctypes.byref(S)))
        return seg[: S.value].copy(), off[: S.value + 1].copy(), rows

    def describe(self) -> list:
        import json

        buf = ctypes.create_string_buffer(8192)
        _check(lib.atmm_plan_describe(self._h, buf, 8192))
        return json.loads(buf.value.decode())

    def stats(self) -> Tuple[int, int, int]:
        a, b, c = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
        _check(lib.atmm_plan_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def apply(self, x, y, layer: int = 0, scale: float = 1.0, stream=None) -> None:
        """y[row] += scale * s_a * (x[row] @ down_a[layer]) @ up_a[layer] (torch CUDA tensors).
        fp32 x and y on a precise registry take the fp32-faithful path."""
        import torch

        if x.dtype == torch.float32 and y.dtype == torch.float32 and self.registry.precise:
            if x.dim() != 2 or y.dim() != 2 or x.shape[0] != self.n or y.shape[0] != self.n:
                raise ShapeError(f"x/y must be 2-D with {self.n} rows")
            if x.stride(1) != 1 or y.stride(1) != 1 or not (x.is_cuda and y.is_cuda):
                raise ShapeError("x and y must be CUDA tensors with contiguous rows")
            _check(lib.atmm_bypass_apply_f32(self._h, layer, x.data_ptr(), x.stride(0), y.data_ptr(), y.stride(0),
                                             float(scale), _stream_ptr(stream)))
            return
        if x.dtype != torch.bfloat16 or not x.is_cuda:
            raise ShapeError("x must be a CUDA bfloat16 tensor")
        if y.dtype not in (torch.bfloat16, torch.float32) or not y.is_cuda:
            raise ShapeError("y must be a CUDA bfloat16 or float32 tensor")
        if x.dim() != 2 or y.dim() != 2 or x.shape[0] != self.n or y.shape[0] != self.n:
            raise ShapeError(f"x/y must be 2-D with {self.n} rows")
        if x.stride(1) != 1 or y.stride(1) != 1:
            raise ShapeError("x and y rows must be contiguous")
        _check(lib.atmm_bypass_apply(self._h, layer, x.data_ptr(), x.stride(0), y.data_ptr(), y.stride(0),
                                     BF16 if y.dtype == torch.bfloat16 else F32, float(scale), _stream_ptr(stream)))

    def apply_group(self, xs, ys, layers, scale: float = 1.0, stream=None) -> None:
        """Independent applications (xs[c], ys[c], layers[c]) in one launch
        where the kernels allow it (include/atmm_b200.h atmm_bypass_apply_group)."""
        import torch

        if not (1 <= len(xs) == len(ys) == len(layers) <= 8):
            raise ConfigError("apply_group takes 1..8 (x, y, layer) calls")
        for x, y in zip(xs, ys):
            if x.dtype != torch.bfloat16 or not x.is_cuda or x.shape != xs[0].shape or x.stride() != xs[0].stride():
                raise ShapeError("every x must be a CUDA bfloat16 tensor of the same shape and strides")
            if y.dtype != ys[0].dtype or not y.is_cuda or y.shape != ys[0].shape or y.stride() != ys[0].stride():
                raise ShapeError("every y must be a CUDA tensor of the same dtype, shape and strides")
        if xs[0].shape[0] != self.n or ys[0].shape[0] != self.n:
            raise ShapeError(f"x/y must be 2-D with {self.n} rows")
        lay = np.asarray(layers, np.int64)
        xp = (ctypes.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
        yp = (ctypes.c_void_p * len(ys))(*[y.data_ptr() for y in ys])
        _check(lib.atmm_bypass_apply_group(self._h, len(xs), _p(lay, i64p), xp, xs[0].stride(0), yp, ys[0].stride(0),
                                           BF16 if ys[0].dtype == torch.bfloat16 else F32, float(scale),
                                           _stream_ptr(stream)))

    def residual_host_bf16(self, x_host: np.ndarray, y_host: np.ndarray, layer: int = 0, scale: float = 1.0,
                           stream=None) -> None:
        """End-to-end: host bf16 (uint16) buffers in, y_host updated in place."""
        if x_host.dtype != np.uint16 or y_host.dtype != np.uint16:
            raise ShapeError("host buffers must be bf16 bit patterns (uint16)")
        if not (x_host.flags.c_contiguous and y_host.flags.c_contiguous):
            raise ShapeError("host buffers must be C-contiguous")
        _check(lib.atmm_bypass_residual_host_bf16(self._h, layer, _p(x_host, u16p), _p(y_host, u16p),
                                                  float(scale), _stream_ptr(stream)))


class MixturePlan:
    """forward_mixture's bypass (model.hpp:252-328) for one layer as ONE fused
    launch: rows assigned to the merged adapter ride the merged weights (no
    bypass); every guest row a gets (x.down_a).up_a - (x.down_m).up_m through
    a combined slot [down_a | down_m], [up_a ; -up_m] (K concatenation), so
    the own branch and the cancel branch are summed in fp32 in TMEM and
    rounded into Y once.  Combined slots are created once per (a, merged)
    pair and cached on the registry (negative ids, never user-visible)."""

    def __init__(self, registry: AdapterRegistry, assignment: Sequence[int], merged_id: int,
                 table: Optional[TilingTable] = None):
        a = _i32(assignment).reshape(-1)
        if merged_id not in registry:
            raise ModeError("mixture integrity: subtraction branch missing (merged adapter not in the registry)")
        combos = registry.__dict__.setdefault("_combined", {})
        guest = np.nonzero(a != merged_id)[0].astype(np.int32)
        fused_rows, fused_virt, two_rows, two_ids = [], [], [], []
        for row in guest:
            key = (int(a[row]), int(merged_id))
            if key not in combos:
                if key[0] not in registry:
                    raise UnknownAdapterError(f"unknown adapter id {key[0]}")
                vid = -(1 << 20) - len(combos)
                try:
                    registry.put_combined(vid, [(key[0], 1.0), (key[1], -1.0)])
                    combos[key] = vid
                except ConfigError:
                    # combined rank above 128 (or a rank-chunked part): these
                    # guests take the two-pass form, own branch then cancel
                    combos[key] = None
            if combos[key] is None:
                two_rows.append(row)
                two_ids.append(key[0])
            else:
                fused_rows.append(row)
                fused_virt.append(combos[key])
        self.n = int(a.size)
        self.guest_rows = guest
        self.plan = (BypassPlan(registry, fused_virt, table, rows=fused_rows, n_rows=self.n)
                     if fused_rows else None)
        self.two_pass_rows = np.asarray(two_rows, np.int32)
        self.own = self.cancel = None
        if two_rows:
            self.own = BypassPlan(registry, two_ids, table, rows=two_rows, n_rows=self.n)
            self.cancel = BypassPlan(registry, [int(merged_id)] * len(two_rows), table, rows=two_rows, n_rows=self.n)

    def apply(self, x, y, layer: int = 0, scale: float = 1.0, stream=None) -> None:
        if self.plan is not None:
            self.plan.apply(x, y, layer, scale, stream)
        if self.own is not None:
            self.own.apply(x, y, layer, scale, stream)
            self.cancel.apply(x, y, layer, -scale, stream)


class GemmOpts(ctypes.Structure):
    """atmm_gemm_opts: explicit GEMM tile options (0 / pair -1 = automatic)."""

    _fields_ = [("pair", ctypes.c_int32), ("bn", ctypes.c_int32), ("kz", ctypes.c_int32), ("ks", ctypes.c_int32),
                ("mc", ctypes.c_int32), ("stages", ctypes.c_int32)]


def _gemm_opts(opts: Optional[dict]):
    if not opts:
        return None
    o = GemmOpts(pair=-1)
    for k, v in opts.items():
        if k not in ("pair", "bn", "kz", "ks", "mc", "stages"):
            raise ConfigError(f"unknown GEMM option {k!r}")
        setattr(o, k, int(v))
    return ctypes.byref(o)


class LayerForward:
    """The serving model's stack forward on device (model.hpp:192-328):
    cur <- tanh(cur @ W_l + bypass_l(cur)) for every layer, the bypass riding
    the base GEMM as extra K blocks of the same tensor-core accumulator.

    plan: a BypassPlan (forward_unmerged), a MixturePlan over merged weights
    (forward_mixture) or None (forward_merged; then n and hidden_dim give
    the shape).  bf16 activations / weights, fp32 accumulation, bf16 out."""

    STATS = ("n", "d", "bn", "tiles", "grid", "ext_blocks", "shrink_items", "shrink_ks", "sorted", "gemm_stages",
             "shrink_stages", "gemm_cta_group", "gemm_split_k")

    def __init__(self, plan=None, n: Optional[int] = None, hidden_dim: Optional[int] = None, device: int = 0,
                 opts: Optional[dict] = None):
        """opts: explicit GEMM tile options {pair, bn, kz, ks, stages}
        (atmm_gemm_opts), automatic when omitted."""
        if isinstance(plan, MixturePlan):
            if plan.own is not None:
                raise ConfigError("the fused layer forward needs every mixture guest in one combined slot "
                                  "(combined rank <= 128); apply the MixturePlan after the base GEMM instead")
            n = plan.n if n is None else n
            if hidden_dim is None and plan.plan is not None:
                hidden_dim = plan.plan.registry.d_in
            plan = plan.plan
        h = ctypes.c_void_p()
        _check(lib.atmm_forward_create_opts(plan.handle if plan is not None else None, int(device), int(n or 0),
                                            int(hidden_dim or 0), _gemm_opts(opts), ctypes.byref(h)))
        self._h = h
        self.plan = plan  # keeps the plan (and its registry) alive
        st = self.stats()
        self.n, self.d = st["n"], st["d"]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # (module globals are None at interpreter exit)
            lib.atmm_forward_destroy(h)
            self._h = None

    def stats(self) -> dict:
        v = np.zeros(len(self.STATS), np.int64)
        _check(lib.atmm_forward_stats(self._h, _p(v, i64p), v.size))
        return {k: int(x) for k, x in zip(self.STATS, v)}

    def run(self, w, x, out=None, num_layers: Optional[int] = None, stream=None):
        """w: [L, d, d] bf16 CUDA tensor (rows contiguous); x: [n, d] bf16 CUDA
        tensor; returns out ([n, d] bf16, allocated when not given)."""
        import torch

        if w.dim() != 3 or w.dtype != torch.bfloat16 or not w.is_cuda or w.stride(2) != 1:
            raise ShapeError("w must be an [L, d, d] bfloat16 CUDA tensor with contiguous rows")
        if x.dim() != 2 or x.dtype != torch.bfloat16 or not x.is_cuda or x.stride(1) != 1:
            raise ShapeError("x must be an [n, d] bfloat16 CUDA tensor with contiguous rows")
        if tuple(x.shape) != (self.n, self.d) or tuple(w.shape[1:]) != (self.d, self.d):
            raise ShapeError(f"x {tuple(x.shape)} / w {tuple(w.shape)} do not match n={self.n}, d={self.d}")
        if out is None:
            out = torch.empty((self.n, self.d), dtype=torch.bfloat16, device=x.device)
        L = w.shape[0] if num_layers is None else int(num_layers)
        _check(lib.atmm_forward_run(self._h, w.data_ptr(), w.stride(1), w.stride(0), L, x.data_ptr(), x.stride(0),
                                    out.data_ptr(), out.stride(0), _stream_ptr(stream)))
        return out


def forward_unmerged(w, x, assignment: Sequence[int], registry: AdapterRegistry, table=None):
    """forward_unmerged (model.hpp:216-246) on device tensors."""
    return LayerForward(BypassPlan(registry, assignment, table)).run(w, x)


def forward_mixture(w_merged, x, assignment: Sequence[int], registry: AdapterRegistry, merged_id: int, table=None):
    """forward_mixture (model.hpp:251-328): w_merged already holds adapter
    merged_id (merge_layers_into); guest rows get own - merged bypass."""
    mp = MixturePlan(registry, assignment, merged_id, table)
    return LayerForward(mp, n=mp.n, hidden_dim=registry.d_in).run(w_merged, x)


def forward_merged(w, x, device: Optional[int] = None):
    """forward_merged (model.hpp:192-211): no bypass."""
    dev = x.device.index if device is None else device
    return LayerForward(None, n=x.shape[0], hidden_dim=x.shape[1], device=dev or 0).run(w, x)


def gemm(a, b, out=None, out_dtype=None, opts: Optional[dict] = None):
    """Plain device GEMM out = a @ b (atmm_multiply_into, atmm.hpp:111-154,
    with a dense right operand; the base GEMM of model.hpp:238): bf16 CUDA
    tensors a [m, k], b [k, n] (unit inner stride), fp32 accumulation, out
    bf16 or fp32 [m, n] (overwritten)."""
    import torch

    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
        raise ShapeError(f"gemm shapes {tuple(a.shape)} x {tuple(b.shape)} do not chain")
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or not (a.is_cuda and b.is_cuda):
        raise ShapeError("a and b must be bf16 CUDA tensors")
    if a.stride(1) != 1 or b.stride(1) != 1:
        raise ShapeError("a and b need unit inner stride")
    m, k = a.shape
    n = b.shape[1]
    if out is None:
        out = torch.empty(m, n, device=a.device, dtype=out_dtype or torch.bfloat16)
    if out.dtype not in (torch.bfloat16, torch.float32) or tuple(out.shape) != (m, n) or out.stride(1) != 1:
        raise ShapeError("out must be a bf16 or fp32 [m, n] tensor with unit inner stride")
    with torch.cuda.device(a.device):
        _check(lib.atmm_gemm_ex(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), out.data_ptr(), out.stride(0),
                                F32 if out.dtype == torch.float32 else BF16, m, k, n, _gemm_opts(opts),
                                torch.cuda.current_stream(a.device).cuda_stream))
    return out


def gemm_f32(a, b, out=None, beta: float = 0.0):
    """fp32-faithful out = a @ b (+ out when beta = 1) on the tensor cores
    (atmm_gemm_f32: one split-bf16 tcgen05 product); fp32 CUDA tensors."""
    import torch

    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
        raise ShapeError(f"gemm shapes {tuple(a.shape)} x {tuple(b.shape)} do not chain")
    if a.dtype != torch.float32 or b.dtype != torch.float32 or not (a.is_cuda and b.is_cuda):
        raise ShapeError("a and b must be fp32 CUDA tensors")
    if a.stride(1) != 1 or b.stride(1) != 1:
        raise ShapeError("a and b need unit inner stride")
    m, k = a.shape
    n = b.shape[1]
    if out is None:
        out = torch.empty(m, n, device=a.device, dtype=torch.float32)
    if out.dtype != torch.float32 or tuple(out.shape) != (m, n) or out.stride(1) != 1:
        raise ShapeError("out must be an fp32 [m, n] tensor with unit inner stride")
    with torch.cuda.device(a.device):
        _check(lib.atmm_gemm_f32(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), out.data_ptr(), out.stride(0),
                                 m, k, n, float(beta), torch.cuda.current_stream(a.device).cuda_stream))
    return out


def forward_f32(w, x, plans=(), out=None, stream=None):
    """The stack forward (model.hpp:192-328) fp32-faithfully:
    cur <- tanh(cur @ W_l + sum_i s_i bypass_{plan_i, l}(cur)); plans is a
    sequence of (BypassPlan on a precise registry, scale)."""
    import torch

    if w.dim() != 3 or w.dtype != torch.float32 or not w.is_cuda or w.stride(2) != 1:
        raise ShapeError("w must be an [L, d, d] fp32 CUDA tensor with contiguous rows")
    if x.dim() != 2 or x.dtype != torch.float32 or not x.is_cuda or x.stride(1) != 1:
        raise ShapeError("x must be an [n, d] fp32 CUDA tensor with contiguous rows")
    n, d = x.shape
    if tuple(w.shape[1:]) != (d, d):
        raise ShapeError(f"w {tuple(w.shape)} does not match d={d}")
    if out is None:
        out = torch.empty(n, d, device=x.device, dtype=torch.float32)
    hs = (ctypes.c_void_p * max(1, len(plans)))(*[p.handle for p, _ in plans])
    sc = _f32([s for _, s in plans] or [0.0])
    _check(lib.atmm_forward_f32(w.data_ptr(), w.stride(1), w.stride(0), w.shape[0], n, d, x.data_ptr(), x.stride(0),
                                out.data_ptr(), out.stride(0), hs, _p(sc, f32p), len(plans), _stream_ptr(stream)))
    return out


def run_bypass_host_bf16_pipelined(plan: "BypassPlan", xs, outs, layers) -> None:
    """run_bypass (batch.hpp:48) end to end from bf16 host buffers (uint16
    numpy views, pinned for overlap): outs[i] = bypass(xs[i]) at layers[i],
    batches pipelined over H2D / compute / D2H."""
    n = len(xs)
    if not (n == len(outs) == len(layers)):
        raise ShapeError("xs, outs and layers must have the same length")
    for a in list(xs) + list(outs):
        if a.dtype != np.uint16 or not a.flags.c_contiguous:
            raise ShapeError("host buffers must be C-contiguous uint16 (bf16 bits)")
    lay = np.asarray(layers, np.int64)
    xp = (ctypes.c_void_p * n)(*[a.ctypes.data for a in xs])
    op = (ctypes.c_void_p * n)(*[a.ctypes.data for a in outs])
    _check(lib.atmm_run_bypass_host_bf16_pipelined(plan.handle, _p(lay, i64p), xp, op, n))


def residual_host_bf16_pipelined(plan: "BypassPlan", xs, ys, layers, scale: float = 1.0) -> None:
    """Serving form: one micro-batch per (x, y) host pair (uint16 bf16 bit
    patterns, pinned for overlap), pipelined H2D / kernel / D2H."""
    count = len(xs)
    if len(ys) != count or len(layers) != count:
        raise ShapeError("xs, ys and layers must have the same length")
    for x, y in zip(xs, ys):
        if x.dtype != np.uint16 or y.dtype != np.uint16 or not (x.flags.c_contiguous and y.flags.c_contiguous):
            raise ShapeError("host buffers must be C-contiguous uint16 (bf16 bit patterns)")
    xp = (ctypes.c_void_p * count)(*[x.ctypes.data for x in xs])
    yp = (ctypes.c_void_p * count)(*[y.ctypes.data for y in ys])
    la = np.ascontiguousarray(np.asarray(layers, np.int64))
    _check(lib.atmm_bypass_residual_host_bf16_pipelined(plan.handle, _p(la, i64p), xp, yp, count, float(scale)))


def run_bypass(registry: AdapterRegistry, x, assignment: Sequence[int], layer: int = 0,
               table: Optional[TilingTable] = None) -> np.ndarray:
    """batch.hpp:48: returns the fresh bypass matrix (host fp32 in/out)."""
    xa = _f32(x)
    a = _i32(assignment).reshape(-1)
    if xa.ndim != 2 or xa.shape[1] != registry.d_in:
        raise ShapeError(f"run_bypass: x must be n x {registry.d_in}")
    if xa.shape[0] != a.size:
        raise ShapeError(f"run_bypass: batch has {xa.shape[0]} rows but plan covers {a.size}")
    out = np.zeros((a.size, registry.d_out), np.float32)
    _check(lib.atmm_run_bypass_host(registry.handle, _p(xa, f32p), a.size, _p(a, i32p), layer,
                                    table.handle if table else None, _p(out, f32p)))
    return out


def delta_w(registry: AdapterRegistry, adapter_id: int, layer: int = 0) -> np.ndarray:
    """model.hpp:130-140: s * down @ up (host fp32)."""
    out = np.zeros((registry.d_in, registry.d_out), np.float32)
    _check(lib.atmm_delta_w_host(registry.handle, adapter_id, layer, _p(out, f32p)))
    return out


def merge_into(registry: AdapterRegistry, adapter_id: int, layer: int, w, sign: float = 1.0, stream=None) -> None:
    """W (+/-)= s * down @ up in place on a CUDA tensor (fp32 or bf16)."""
    import torch

    if w.dim() != 2 or w.stride(1) != 1 or not w.is_cuda or w.dtype not in (torch.float32, torch.bfloat16):
        raise ShapeError("w must be a row-contiguous 2-D CUDA float32/bfloat16 tensor")
    if tuple(w.shape) != (registry.d_in, registry.d_out):
        raise ShapeError(f"w shape {tuple(w.shape)} != ({registry.d_in}, {registry.d_out})")
    _check(lib.atmm_merge_apply(registry.handle, adapter_id, layer, w.data_ptr(), w.stride(0),
                                F32 if w.dtype == torch.float32 else BF16, float(sign), _stream_ptr(stream)))


def merge_layers_into(registry: AdapterRegistry, adapter_id: int, w, sign: float = 1.0, layer0: int = 0,
                      stream=None) -> None:
    """W[l] (+/-)= s * down[layer0 + l] @ up[layer0 + l] for every layer of a
    [L, d_in, d_out] CUDA tensor in ONE launch (the mode switch's merge of
    all layers, model.hpp:144-188)."""
    import torch

    if w.dim() != 3 or w.stride(2) != 1 or not w.is_cuda or w.dtype not in (torch.float32, torch.bfloat16):
        raise ShapeError("w must be a [L, d_in, d_out] CUDA float32/bfloat16 tensor with contiguous rows")
    if tuple(w.shape[1:]) != (registry.d_in, registry.d_out):
        raise ShapeError(f"w shape {tuple(w.shape)} != (L, {registry.d_in}, {registry.d_out})")
    _check(lib.atmm_merge_apply_layers(registry.handle, adapter_id, layer0, w.shape[0], w.data_ptr(), w.stride(1),
                                       w.stride(0), F32 if w.dtype == torch.float32 else BF16, float(sign),
                                       _stream_ptr(stream)))


UNMERGED, MERGED, MIXTURE = 0, 1, 2
_MODE_NAMES = {UNMERGED: "unmerged", MERGED: "merged", MIXTURE: "mixture"}


class ModelState:
    """ModelState (model.hpp:104-112) bound to a model's device weights
    ``w`` ([L, d_in, d_out] CUDA tensor, fp32 or bf16, address-stable): merge
    / unmerge enforce the reference's mode contract (ModeError on a double
    merge or an unmerge of the wrong adapter, model.hpp:147,170,173), every
    weight rewrite is ONE all-layer launch, and mode_switch issues the minimal
    sequence (serving.hpp:38-74)."""

    def __init__(self, registry: AdapterRegistry, w):
        import torch

        if w.dim() != 3 or w.stride(2) != 1 or not w.is_cuda or w.dtype not in (torch.float32, torch.bfloat16):
            raise ShapeError("w must be a [L, d_in, d_out] CUDA float32/bfloat16 tensor with contiguous rows")
        if tuple(w.shape) != (registry.num_layers, registry.d_in, registry.d_out):
            raise ShapeError(f"w shape {tuple(w.shape)} != ({registry.num_layers}, {registry.d_in}, {registry.d_out})")
        h = ctypes.c_void_p()
        _check(lib.atmm_state_create(registry.handle, w.data_ptr(), w.stride(1), w.stride(0),
                                     F32 if w.dtype == torch.float32 else BF16, ctypes.byref(h)))
        self._h = h
        self.registry = registry
        self.w = w  # keeps the bound weights alive

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # (module globals are None at interpreter exit)
            lib.atmm_state_destroy(h)
            self._h = None

    def _get(self):
        m, a, n = ctypes.c_int(0), ctypes.c_int32(0), ctypes.c_int64(0)
        _check(lib.atmm_state_get(self._h, ctypes.byref(m), ctypes.byref(a), ctypes.byref(n)))
        return m.value, a.value, n.value

    @property
    def mode(self) -> str:
        return _MODE_NAMES[self._get()[0]]

    @property
    def merged_adapter(self) -> int:
        return self._get()[1]

    @property
    def weight_writes(self) -> int:
        return self._get()[2]

    def merge(self, adapter_id: int, stream=None) -> None:
        _check(lib.atmm_state_merge(self._h, int(adapter_id), _stream_ptr(stream)))

    def unmerge(self, adapter_id: int, stream=None) -> None:
        _check(lib.atmm_state_unmerge(self._h, int(adapter_id), _stream_ptr(stream)))

    def set_mixture(self, adapter_id: int) -> None:
        _check(lib.atmm_state_set_mixture(self._h, int(adapter_id)))

    def mode_switch(self, to_mode: str, target_adapter: int = -1, stream=None) -> int:
        """Returns the number of all-layer weight rewrites issued (0 for
        merged <-> mixture of the same adapter)."""
        m = {v: k for k, v in _MODE_NAMES.items()}[to_mode]
        n = ctypes.c_int64(0)
        _check(lib.atmm_state_mode_switch(self._h, m, int(target_adapter), _stream_ptr(stream), ctypes.byref(n)))
        return n.value


def save_matrix(path: str, m) -> None:
    """save_matrix<float> (matrix.hpp:183-196): the reference's binary format."""
    a = _f32(m)
    if a.ndim != 2:
        raise ShapeError("save_matrix takes a 2-D matrix")
    _check(lib.atmm_matrix_save(str(path).encode(), a.shape[0], a.shape[1], _p(a, f32p)))


def load_matrix(path: str) -> np.ndarray:
    """load_matrix<float> (matrix.hpp:198-218)."""
    r, c = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib.atmm_matrix_load(str(path).encode(), ctypes.byref(r), ctypes.byref(c), None, 0))
    out = np.zeros((r.value, c.value), np.float32)
    _check(lib.atmm_matrix_load(str(path).encode(), ctypes.byref(r), ctypes.byref(c), _p(out, f32p), out.size))
    return out


def fixture_info(directory: str) -> dict:
    """manifest.json of a reference fixture: layers, hidden dim, adapter ids / ranks."""
    L, d, n = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib.atmm_fixture_info(str(directory).encode(), ctypes.byref(L), ctypes.byref(d), ctypes.byref(n), None,
                                 None, 0))
    ids = np.zeros(n.value, np.int32)
    ranks = np.zeros(n.value, np.int64)
    _check(lib.atmm_fixture_info(str(directory).encode(), ctypes.byref(L), ctypes.byref(d), ctypes.byref(n),
                                 _p(ids, i32p), _p(ranks, i64p), n.value))
    return {"num_layers": L.value, "hidden_dim": d.value, "adapters": dict(zip(ids.tolist(), ranks.tolist()))}


def atmm_multiply(a, b, config: Sequence[int]) -> np.ndarray:
    """atmm.hpp:144-154 (host fp32 in/out, bf16 tcgen05 compute)."""
    aa, bb = _f32(a), _f32(b)
    if aa.ndim != 2 or bb.ndim != 2 or aa.shape[1] != bb.shape[0]:
        raise ShapeError(f"atmm_multiply: shape mismatch {aa.shape[0]}x{aa.shape[1]} vs {bb.shape[0]}x{bb.shape[1]}")
    m, k = aa.shape
    n = bb.shape[1]
    out = np.zeros((m, n), np.float32)
    _check(lib.atmm_multiply_host(_p(aa, f32p), m, k, _p(bb, f32p), n, _p(out, f32p), _p(_i32(config), i32p)))
    return out


# ------------------------------------------------- offline tiling search ---


class TuneShape(ctypes.Structure):
    """atmm_tune_shape: `segments` segments of `m` rows, each its own adapter
    of rank `rank`, at (d_in, d_out) (the B200 re-reading of GemmShape,
    atmm.hpp:218-220)."""

    _fields_ = [("m", ctypes.c_int64), ("d_in", ctypes.c_int64), ("rank", ctypes.c_int64),
                ("d_out", ctypes.c_int64), ("segments", ctypes.c_int64)]

    def as_tuple(self) -> Tuple[int, int, int, int, int]:
        return (self.m, self.d_in, self.rank, self.d_out, self.segments)


def _shapes(shapes) -> ctypes.Array:
    arr = (TuneShape * len(shapes))()
    for i, sh in enumerate(shapes):
        arr[i] = sh if isinstance(sh, TuneShape) else TuneShape(*[int(v) for v in sh])
    return arr


def _launches(launches) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate([_launch5(l) for l in launches]))


_DEFAULT_TABLE = {}
DEFAULT_TABLE_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tables", "b200_tiling_table.json")


def default_table() -> Optional["TilingTable"]:
    """The packaged B200-profiled tiling table (tools/tune.py: tiling_search
    over default_shape_grid + the benched batch shapes), loaded once; None
    when the package ships without one (the built-in heuristic applies)."""
    if "t" not in _DEFAULT_TABLE:
        _DEFAULT_TABLE["t"] = TilingTable.load(DEFAULT_TABLE_PATH) if os.path.exists(DEFAULT_TABLE_PATH) else None
    return _DEFAULT_TABLE["t"]


def default_shape_grid(d_in: int, d_out: Optional[int] = None, ranks: Optional[Sequence[int]] = None) -> List[tuple]:
    """default_shape_grid (atmm.hpp:341-355) for the bypass: (m, d_in, rank, d_out, segments) tuples."""
    d_out = d_in if d_out is None else d_out
    rk = np.ascontiguousarray(np.asarray(ranks or [], np.int64))
    n = ctypes.c_int64(0)
    _check(lib.atmm_default_shape_grid(d_in, d_out, _p(rk, i64p) if rk.size else None, rk.size, None, 0,
                                       ctypes.byref(n)))
    arr = (TuneShape * n.value)()
    _check(lib.atmm_default_shape_grid(d_in, d_out, _p(rk, i64p) if rk.size else None, rk.size, arr, n.value,
                                       ctypes.byref(n)))
    return [a.as_tuple() for a in arr]


def default_launch_candidates() -> List[Tuple[int, ...]]:
    """The curated B200 candidate launches {tile_m, cluster, bn, stages, path}."""
    n = ctypes.c_int64(0)
    _check(lib.atmm_default_launch_candidates(None, 0, ctypes.byref(n)))
    out = np.zeros(5 * n.value, np.int32)
    _check(lib.atmm_default_launch_candidates(_p(out, i32p), n.value, ctypes.byref(n)))
    return [tuple(int(v) for v in out[5 * i: 5 * i + 5]) for i in range(n.value)]


def benchmark_launch(shape, launch: Sequence[int], trials: int = 5, seed: int = 0x5EEDBEEF, device: int = 0) -> int:
    """benchmark_config (atmm.hpp:188-216): median ns per apply."""
    sh = _shapes([shape])
    out = ctypes.c_int64(0)
    _check(lib.atmm_benchmark_launch(device, sh, _p(_launch5(launch), i32p), int(trials), int(seed), ctypes.byref(out)))
    return out.value


def grid_bench_ns(shapes, launches, trials: int = 5, rounds: int = 3, device: int = 0,
                  failures: Optional[list] = None) -> np.ndarray:
    """grid_bench_ns (atmm.hpp:229-270): [shapes x launches] median-of-round-medians ns."""
    sh, la = _shapes(shapes), _launches(launches)
    scores = np.zeros((len(shapes), len(launches)), np.int64)
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib.atmm_grid_bench_ns(device, sh, len(shapes), _p(la, i32p), len(launches), int(trials), int(rounds),
                                  _p(scores, i64p), buf, len(buf)))
    if failures is not None:
        failures.extend(x for x in buf.value.decode().split("\n") if x)
    return scores


def table_from_scores(shapes, launches, scores, failures: Optional[list] = None) -> "TilingTable":
    """The selection half of tiling_search (atmm.hpp:293-329) over a score
    grid [shapes x launches] (np.iinfo(np.int64).max = failed).  Host only."""
    sh, la = _shapes(shapes), _launches(launches)
    sc = np.ascontiguousarray(np.asarray(scores, np.int64))
    if sc.shape != (len(shapes), len(launches)):
        raise ShapeError("scores must be [len(shapes), len(launches)]")
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib.atmm_table_from_scores(sh, len(shapes), _p(la, i32p), len(launches), _p(sc, i64p), ctypes.byref(h),
                                      buf, len(buf)))
    if failures is not None:
        failures.extend(x for x in buf.value.decode().split("\n") if x)
    return TilingTable(_handle=h)


def tiling_search(shapes, launches=None, trials: int = 5, device: int = 0,
                  failures: Optional[list] = None) -> "TilingTable":
    """tiling_search (atmm.hpp:276-330) on the B200: per-shape argmin, the
    most frequent winner as default; returns a TilingTable (save() writes the
    reference's JSON schema plus the "sm100" launch extension)."""
    launches = launches or default_launch_candidates()
    sh, la = _shapes(shapes), _launches(launches)
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib.atmm_tiling_search(device, sh, len(shapes), _p(la, i32p), len(launches), int(trials), ctypes.byref(h),
                                  buf, len(buf)))
    if failures is not None:
        failures.extend(x for x in buf.value.decode().split("\n") if x)
    return TilingTable(_handle=h)


def shard_rows(assignment: Sequence[int], adapter_ranks: dict, d_in: int, d_out: int, num_shards: int) -> np.ndarray:
    """LPT request sharding over GPUs; returns shard index per row."""
    a = _i32(assignment).reshape(-1)
    ids = _i32(sorted(adapter_ranks))
    ranks = np.ascontiguousarray(np.asarray([adapter_ranks[i] for i in sorted(adapter_ranks)], np.int64))
    out = np.zeros(a.size, np.int32)
    _check(lib.atmm_shard_rows(_p(a, i32p), a.size, _p(ids, i32p), _p(ranks, i64p), ids.size, d_in, d_out,
                               num_shards, _p(out, i32p)))
    return out
