"""Synthetic ATMM workloads at the BASELINE.json configurations.

Shapes follow SURVEY.md sec. 8(d): contiguous per-adapter runs of rows that
are then shuffled (so the kernel's row gather is exercised), Zipf segment
lengths for the adaptive-tiling stress case, factors ~ U(+-1/sqrt(r)) like
LoraAdapter::random (adapter.hpp:53-73), activations ~ U(-1, 1).
Data is synthetic (there is no network for checkpoints).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List

import numpy as np


@dataclass
class BypassWorkload:
    name: str
    d_in: int
    d_out: int
    tokens: int
    ranks: Dict[int, int]                 # adapter id -> rank
    lengths: Dict[int, int]               # adapter id -> segment rows
    assignment: np.ndarray = field(repr=False, default=None)

    @property
    def adapters(self) -> List[int]:
        return sorted(self.ranks)

    def flops(self) -> int:
        """Algorithmic FLOPs, flops.hpp / batch.hpp:45-47: sum_seg 2*ns*r*(d_in + d_out)."""
        return int(sum(2 * self.lengths[a] * self.ranks[a] * (self.d_in + self.d_out) for a in self.ranks))

    def bytes(self, y_bytes: int = 2) -> int:
        """Algorithmic HBM bytes of the fused op: X read, Y read + write, factors once (bf16)."""
        used = [a for a in self.ranks if self.lengths[a] > 0]
        factors = sum((self.d_in + self.d_out) * self.ranks[a] * 2 for a in used)
        return int(self.tokens * self.d_in * 2 + self.tokens * self.d_out * 2 * y_bytes + factors)


def equal_lengths(tokens: int, ids: List[int]) -> Dict[int, int]:
    base = tokens // len(ids)
    out = {a: base for a in ids}
    out[ids[0]] += tokens - base * len(ids)
    return out


def zipf_lengths(tokens: int, ids: List[int]) -> Dict[int, int]:
    """n_i = floor(tokens * (1/(i+1)) / H_A), remainder to adapter 0."""
    A = len(ids)
    H = sum(1.0 / (i + 1) for i in range(A))
    out = {a: int(np.floor(tokens * (1.0 / (i + 1)) / H)) for i, a in enumerate(ids)}
    out[ids[0]] += tokens - sum(out.values())
    return out


def make_assignment(lengths: Dict[int, int], seed: int = 3, shuffle: bool = True) -> np.ndarray:
    rows = np.concatenate([np.full(lengths[a], a, np.int32) for a in sorted(lengths)])
    if shuffle:
        rows = rows[np.random.default_rng(seed).permutation(rows.size)]
    return np.ascontiguousarray(rows, np.int32)


def bypass_config(name: str, seed: int = 3) -> BypassWorkload:
    """cfg1, cfg2, cfg3, cfg5 of BASELINE.json (cfg4 is the merge, see merge_config)."""
    if name == "cfg1":
        ids = list(range(4))
        w = BypassWorkload(name, 4096, 4096, 64, {a: 16 for a in ids}, equal_lengths(64, ids))
    elif name == "cfg2":
        ids = list(range(16))
        w = BypassWorkload(name, 4096, 4096, 512, {a: 16 for a in ids}, equal_lengths(512, ids))
    elif name == "cfg3":
        ids = list(range(32))
        ranks = {a: (8, 16, 32, 64)[a % 4] for a in ids}
        w = BypassWorkload(name, 4096, 4096, 2048, ranks, zipf_lengths(2048, ids))
    elif name == "cfg5":
        ids = list(range(64))
        w = BypassWorkload(name, 5120, 5120, 8192, {a: 64 for a in ids}, equal_lengths(8192, ids))
    elif name == "paper_in1":  # the paper's ATMM Input 1: 256 x 4096 . 4096 x 32
        w = BypassWorkload(name, 4096, 4096, 256, {0: 32}, {0: 256})
    elif name == "paper_in2":  # the paper's ATMM Input 2: 8192 x 4096 . 4096 x 128
        w = BypassWorkload(name, 4096, 4096, 8192, {0: 128}, {0: 8192})
    elif name == "cfg5_r16":
        ids = list(range(64))
        w = BypassWorkload(name, 5120, 5120, 8192, {a: 16 for a in ids}, equal_lengths(8192, ids))
    else:
        raise KeyError(name)
    w.assignment = make_assignment(w.lengths, seed)
    return w


@dataclass
class MergeWorkload:
    name: str = "cfg4"
    d_in: int = 4096
    d_out: int = 11008
    rank: int = 64
    layers: int = 32

    def flops(self, w_bytes: int = 2) -> int:
        """Per layer: 2*d_in*d_out*r (dW) + d_in*d_out (the add)."""
        return int(self.layers * (2 * self.d_in * self.d_out * self.rank + self.d_in * self.d_out))

    def bytes(self, w_bytes: int = 2) -> int:
        """Per layer: W read + write, factors once."""
        return int(self.layers * (2 * self.d_in * self.d_out * w_bytes + (self.d_in + self.d_out) * self.rank * 2))


def random_factors(rng: np.random.Generator, d_in: int, d_out: int, rank: int, layers: int = 1):
    s = 1.0 / np.sqrt(np.float32(rank))
    down = rng.uniform(-s, s, size=(layers, d_in, rank)).astype(np.float32)
    up = rng.uniform(-s, s, size=(layers, rank, d_out)).astype(np.float32)
    return down, up
