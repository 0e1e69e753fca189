"""Request sharding of one ATMM batch over the GPUs of a node.

Every segment (the rows of one adapter) depends only on its own X rows and its
adapter's factors, and output rows are disjoint (run_bypass, batch.hpp:57-79),
so the batch shards by request with no collective on the data path: each rank
runs the fused bypass on the rows of its shard, with only the adapters its
shard touches resident.  Placement is longest-processing-time over whole
segments (atmm_shard_rows in the C ABI; cost = bytes the segment moves), so
it is deterministic and every rank computes the same plan without
communicating.

`ShardedBypass` is one rank's launcher: registry of the shard's adapters, a
plan over the shard's rows, and two ways to run it --
  * apply_local(x_local, y_local): X / Y hold only the shard's rows (in
    ascending global row order), the serving layout where each GPU receives
    its own requests;
  * apply_global(x, y): X / Y are the whole batch on this device; the plan is
    row-mapped (atmm_plan_create_mapped), so the kernels read and write the
    shard's rows in place (no staging copy).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from .atmm import shard_rows


@dataclass
class Shard:
    rank: int
    rows: np.ndarray          # batch rows owned by this rank (ascending)
    assignment: np.ndarray    # adapter id per owned row
    adapters: List[int]       # adapters this rank must hold


def shard_batch(assignment, ranks: Dict[int, int], d_in: int, d_out: int, world: int) -> List[Shard]:
    a = np.ascontiguousarray(np.asarray(assignment, np.int32))
    owner = shard_rows(a, ranks, d_in, d_out, world)
    shards = []
    for r in range(world):
        rows = np.nonzero(owner == r)[0].astype(np.int64)
        sub = a[rows]
        shards.append(Shard(r, rows, sub, sorted(set(int(v) for v in sub))))
    return shards


def shard_cost(shard: Shard, ranks: Dict[int, int], d_in: int, d_out: int) -> float:
    """Bytes the shard moves (X read, Y read + write, factors once), bf16."""
    rows = float(shard.rows.size)
    return rows * (2.0 * d_in + 4.0 * d_out) + sum(2.0 * ranks[a] * (d_in + d_out) for a in shard.adapters)


def shard_flops(shard: Shard, ranks: Dict[int, int], d_in: int, d_out: int) -> int:
    """Algorithmic FLOPs of the shard (flops.hpp: sum_seg 2*ns*r*(d_in + d_out))."""
    ids, counts = np.unique(shard.assignment, return_counts=True)
    return int(sum(2 * int(c) * ranks[int(a)] * (d_in + d_out) for a, c in zip(ids, counts)))


def replicate_batch(assignment, ranks: Dict[int, int], copies: int) -> Tuple[np.ndarray, Dict[int, int]]:
    """`copies` independent request batches of the same shape as ONE global
    batch (weak scaling): copy c's adapter ids are offset by c * (max id + 1)
    and its rows follow copy c-1's."""
    a = np.asarray(assignment, np.int32)
    stride = int(max(ranks)) + 1
    glob = np.concatenate([a + c * stride for c in range(copies)]).astype(np.int32)
    granks = {int(k) + c * stride: int(v) for c in range(copies) for k, v in ranks.items()}
    return glob, granks


class ShardedBypass:
    """One rank's part of a request-sharded bypass.

    factors(adapter_id) -> (down [L, d_in, r], up [L, r, d_out]) host fp32 (or
    bf16-exact fp32) arrays; only the shard's adapters are requested and
    uploaded.  Every rank builds the same shard plan from the same inputs."""

    def __init__(self, assignment: Sequence[int], ranks: Dict[int, int], d_in: int, d_out: int, world: int, rank: int,
                 factors: Callable[[int], Tuple[np.ndarray, np.ndarray]], num_layers: int = 1, device: int = 0,
                 scales: Optional[Dict[int, float]] = None, table=None):
        from .atmm import AdapterRegistry, BypassPlan

        if not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside world {world}")
        self.assignment = np.ascontiguousarray(np.asarray(assignment, np.int32))
        self.n = int(self.assignment.size)
        self.ranks = {int(k): int(v) for k, v in ranks.items()}
        self.d_in, self.d_out, self.world, self.rank = d_in, d_out, world, rank
        self.shards = shard_batch(self.assignment, self.ranks, d_in, d_out, world)
        self.shard = self.shards[rank]
        self.device = device
        self.registry = AdapterRegistry(num_layers, d_in, d_out, device=device)
        for a in self.shard.adapters:
            down, up = factors(a)
            self.registry.put(a, down, up, scale=(scales or {}).get(a, 1.0))
        self.table = table
        self.plan = BypassPlan(self.registry, self.shard.assignment, table) if self.shard.rows.size else None
        self._mapped = None

    @property
    def rows(self) -> np.ndarray:
        return self.shard.rows

    def flops(self) -> int:
        return shard_flops(self.shard, self.ranks, self.d_in, self.d_out)

    def bytes(self) -> float:
        return shard_cost(self.shard, self.ranks, self.d_in, self.d_out)

    def apply_local(self, x_local, y_local, layer: int = 0, scale: float = 1.0, stream=None) -> None:
        """y_local[i] += scale * bypass(x_local[i]) for the shard's rows
        (x_local / y_local: [len(rows), d] CUDA tensors in ascending global row order)."""
        if self.plan is None:
            return
        self.plan.apply(x_local, y_local, layer=layer, scale=scale, stream=stream)

    def apply_global(self, x, y, layer: int = 0, scale: float = 1.0, stream=None) -> None:
        """The shard's rows of the whole-batch x / y ([n, d] on this device),
        in place through a row-mapped plan."""
        if self.plan is None:
            return
        if self._mapped is None:
            from .atmm import BypassPlan

            self._mapped = BypassPlan(self.registry, self.shard.assignment, self.table, rows=self.shard.rows,
                                      n_rows=self.n)
        self._mapped.apply(x, y, layer=layer, scale=scale, stream=stream)
