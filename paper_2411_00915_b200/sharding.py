"""Request sharding of one ATMM batch over the GPUs of a node.

Every segment (the rows of one adapter) depends only on its own X rows and its
adapter's factors, and output rows are disjoint, so the batch shards by
request with no collective on the data path: each rank runs the fused bypass
on the rows of its shard, with only the adapters its shard touches resident.
Placement is longest-processing-time over whole segments (atmm_shard_rows in
the C ABI; cost = bytes the segment moves), so it is deterministic and every
rank computes the same plan without communicating.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List

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
