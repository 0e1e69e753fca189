"""CPU, world_size 2 over gloo: the request-sharded multi-GPU path.

Each rank derives its shard of the batch locally (no communication on the
data path); the test all-gathers what every rank decided and checks that the
ranks agree, that the shards partition the batch exactly once with whole
segments, and that the max-over-ranks timing reduction works.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_00915_b200.sharding import shard_batch
        from paper_2411_00915_b200.workloads import bypass_config

        w = bypass_config(cfg)
        shards = shard_batch(w.assignment, w.ranks, w.d_in, w.d_out, world)
        mine = shards[rank]
        # every rank's view of every shard, gathered
        gathered = [None] * world
        dist.all_gather_object(gathered, [s.rows.tolist() for s in shards])
        rows_of_mine = [None] * world
        dist.all_gather_object(rows_of_mine, mine.rows.tolist())
        # max over ranks of a per-rank "time" (the bench's reduction)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, gathered, rows_of_mine, float(t.item()), w.tokens, {int(k): int(v) for k, v in w.lengths.items()},
               w.assignment.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg5"])
def test_request_sharding_two_ranks(cfg):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort(key=lambda r: r[0])
    views = [r[1] for r in results]
    assert views[0] == views[1]  # identical plans on both ranks, no communication needed
    owned = results[0][2]
    tokens, lengths, assignment = results[0][4], results[0][5], np.asarray(results[0][6])
    allrows = sorted(owned[0] + owned[1])
    assert allrows == list(range(tokens))
    for r in range(world):
        ids = set(assignment[owned[r]].tolist())
        for a in ids:
            assert np.count_nonzero(assignment[owned[r]] == a) == lengths[a]
    assert results[0][3] == results[1][3] == float(world)


def test_weak_scaling_batch_shards_evenly():
    """bench.py --gpus N (weak scaling): N copies of a batch with distinct
    adapters shard into N shards of exactly one batch each (LPT, host only)."""
    from paper_2411_00915_b200.sharding import replicate_batch, shard_batch, shard_flops
    from paper_2411_00915_b200.workloads import bypass_config

    for name in ("cfg2", "cfg5"):
        w = bypass_config(name)
        for n in (1, 2, 4, 8):
            glob, granks = replicate_batch(w.assignment, w.ranks, n)
            shards = shard_batch(glob, granks, w.d_in, w.d_out, n)
            assert sorted(s.rows.size for s in shards) == [w.tokens] * n
            assert all(len(s.adapters) == len(w.ranks) for s in shards)
            assert sum(shard_flops(s, granks, w.d_in, w.d_out) for s in shards) == n * w.flops()


def test_strong_scaling_shards_balance_cfg5():
    """bench.py --strong: cfg5 (64 equal segments) split 2/4/8 ways is exact."""
    from paper_2411_00915_b200.sharding import shard_batch
    from paper_2411_00915_b200.workloads import bypass_config

    w = bypass_config("cfg5")
    for n in (2, 4, 8):
        shards = shard_batch(w.assignment, w.ranks, w.d_in, w.d_out, n)
        assert [s.rows.size for s in shards] == [w.tokens // n] * n
