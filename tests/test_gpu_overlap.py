"""Programmatic-dependency elision of the all-to-all bypass (device.cu
pdl_can_elide, kernels.cu wait-before-trigger protocol).

An apply starts its X / Y loads under the preceding launch only when that
launch is an all-to-all bypass touching disjoint bytes.  These tests pin the
decision (launch counters) and the results: every sequence gives the same bits
as the same sequence with ATMM_PLAN_NO_OVERLAP (full dependency), including
the hazards the check must refuse -- Y_i feeding X_i+1 (RAW), Y_i+1 = X_i
(WAR), Y_i+1 = Y_i (WAW) -- eager and under CUDA-graph capture, with a
foreign (non-PDL) kernel in between, and against the oracle.
"""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu

D = 1024
RANKS = {a: 16 for a in range(8)}
ROWS = 24  # rows per adapter: one a2a tile each


def _setup(atmm, oracle, seed=5):
    import torch

    reg = atmm.AdapterRegistry(1, D, D)
    facs = {}
    rng = oracle.rng(seed)
    for a, r in RANKS.items():
        s = 1.0 / np.sqrt(np.float32(r))
        down = oracle.round_bf16(oracle.random_matrix(rng, D, r, -s, s))
        up = oracle.round_bf16(oracle.random_matrix(rng, r, D, -s, s))
        reg.put(a, down[None], up[None])
        facs[a] = (down, up)
    assignment = np.repeat(np.asarray(sorted(RANKS), np.int32), ROWS)
    assignment = assignment[np.random.default_rng(seed).permutation(assignment.size)]
    plan = atmm.BypassPlan(reg, assignment)
    ref_plan = atmm.BypassPlan(reg, assignment)
    ref_plan.set_overlap(False)
    assert [g["path_bf16"] for g in plan.describe()] == ["a2a"]
    n = assignment.size
    bufs = [torch.empty(n, D, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1) for _ in range(8)]
    return reg, facs, assignment, plan, ref_plan, bufs


def _run(plan, bufs, steps, stream):
    """steps: (x index, y index) per apply, on one stream."""
    import torch

    with torch.cuda.stream(stream):
        for xi, yi in steps:
            plan.apply(bufs[xi], bufs[yi], stream=stream)
    stream.synchronize()


def _compare(atmm, plan, ref_plan, bufs, steps):
    import torch

    a = [b.clone() for b in bufs]
    b = [b.clone() for b in bufs]
    s = torch.cuda.Stream()
    before = atmm.overlap_stats()
    _run(plan, a, steps, s)
    mid = atmm.overlap_stats()
    _run(ref_plan, b, steps, s)
    after = atmm.overlap_stats()
    for i, (u, v) in enumerate(zip(a, b)):
        assert torch.equal(u, v), f"buffer {i} differs from the full-dependency run"
    assert after[1] == mid[1], "a NO_OVERLAP plan started early"
    return mid[0] - before[0], mid[1] - before[1], a


def test_independent_batches_start_early_same_bits(gpu, atmm, oracle):
    _, _, _, plan, ref_plan, bufs = _setup(atmm, oracle)
    steps = [(0, 1), (2, 3), (4, 5), (6, 7), (0, 3)]  # the last reads X0 (not written by (6, 7))
    launches, early = _compare(atmm, plan, ref_plan, bufs, steps)[:2]
    assert launches == len(steps)
    assert early >= len(steps) - 1, (launches, early)


def test_dependent_chain_keeps_the_dependency(gpu, atmm, oracle):
    _, facs, assignment, plan, ref_plan, bufs = _setup(atmm, oracle)
    steps = [(0, 1), (1, 2), (2, 3), (3, 4)]  # Y_i is X_i+1 (RAW)
    x0 = bufs[0].float().cpu().numpy()
    launches, early, out = _compare(atmm, plan, ref_plan, bufs, steps)
    assert early == 0 or (early == 1 and launches == len(steps)), (launches, early)
    # the first step against the oracle (the rest chain bf16 outputs)
    want = bufs[1].float().cpu().numpy().astype(np.float64) + oracle.bypass_rows_f64(x0, assignment, facs)
    got = out[1].float().cpu().numpy()
    assert np.max(np.abs(got - want)) <= tol_for(want)


@pytest.mark.parametrize("steps", [
    [(0, 1), (2, 0)],          # WAR: the second writes what the first reads
    [(0, 1), (2, 1)],          # WAW: both accumulate into Y1
    [(0, 1), (1, 1)],          # in place after a write
    [(0, 1), (1, 2), (3, 1)],  # RAW then WAW
])
def test_hazards_are_refused(gpu, atmm, oracle, steps):
    _, _, _, plan, ref_plan, bufs = _setup(atmm, oracle)
    s = __import__("torch").cuda.Stream()
    _run(plan, [b.clone() for b in bufs], [(4, 5)], s)  # a disjoint predecessor on this stream
    before = atmm.overlap_stats()
    a = [b.clone() for b in bufs]
    _run(plan, a, steps, s)
    after = atmm.overlap_stats()
    # the first step follows (4, 5): disjoint, may start early; none of the others may
    assert after[1] - before[1] <= 1, steps
    b = [b.clone() for b in bufs]
    _run(ref_plan, b, steps, s)
    for u, v in zip(a, b):
        assert __import__("torch").equal(u, v)


def test_graph_capture_overlap_same_bits(gpu, atmm, oracle):
    import torch

    _, _, _, plan, ref_plan, bufs = _setup(atmm, oracle)
    steps = [(0, 1), (2, 3), (4, 5), (6, 7), (1, 2), (3, 4)]  # (1, 2) reads Y of step 0 (not the predecessor)
    res = []
    for p in (plan, ref_plan):
        work = [b.clone() for b in bufs]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            p.apply(work[0], work[1], stream=s)  # warm-up (maps, attributes) outside the capture
        s.synchronize()
        work = [b.clone() for b in bufs]
        g = torch.cuda.CUDAGraph()
        before = atmm.overlap_stats()
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            for xi, yi in steps:
                p.apply(work[xi], work[yi], stream=s)
        after = atmm.overlap_stats()
        if p is plan:
            # first captured node has no predecessor; (1, 2) follows (6, 7): disjoint; (3, 4) follows (1, 2): disjoint
            assert after[1] - before[1] == len(steps) - 1, (before, after)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        res.append(work)
    for u, v in zip(*res):
        assert torch.equal(u, v)


def test_foreign_kernel_between_applies(gpu, atmm, oracle):
    """A torch kernel (no PDL attribute) writing the next X between two applies."""
    import torch

    _, _, _, plan, ref_plan, bufs = _setup(atmm, oracle)
    res = []
    for p in (plan, ref_plan):
        work = [b.clone() for b in bufs]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for i in range(4):
                p.apply(work[2 * i], work[2 * i + 1], stream=s)
                if i < 3:
                    work[2 * i + 2].copy_(work[2 * i + 1] * 0.5)  # next X from this Y, by torch
        s.synchronize()
        res.append(work)
    for u, v in zip(*res):
        assert torch.equal(u, v)


def test_two_streams_interleaved(gpu, atmm, oracle):
    """Records are per stream: interleaved applies on two streams (each its
    own chain of disjoint and dependent steps) equal the full-dependency bits."""
    import torch

    _, _, _, plan, ref_plan, bufs = _setup(atmm, oracle)
    res = []
    for p in (plan, ref_plan):
        work = [b.clone() for b in bufs]
        sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
        for i in range(4):
            with torch.cuda.stream(sa):
                p.apply(work[0], work[1 + (i % 2)], stream=sa)      # A: X0 -> Y1 / Y2
            with torch.cuda.stream(sb):
                p.apply(work[4 + (i % 2)], work[6], stream=sb)      # B: X4 / X5 -> Y6
                p.apply(work[6], work[7], stream=sb)                # B: dependent on the previous
        torch.cuda.synchronize()
        res.append(work)
    for u, v in zip(*res):
        assert torch.equal(u, v)


def test_grouped_launches_overlap_same_bits(gpu, atmm, oracle):
    """Grouped applies (one launch, several (X, Y) calls sharing X, like the
    q / k / v projections) overlap the next group only when disjoint."""
    import torch

    _, _, _, plan, ref_plan, bufs = _setup(atmm, oracle)
    groups = [((0, 1), (0, 2), (0, 3)), ((4, 5), (4, 6), (4, 7)),  # disjoint from the first
              ((1, 5), (2, 6), (3, 7))]                            # reads the first group's outputs
    res, early = [], []
    for p in (plan, ref_plan):
        work = [b.clone() for b in bufs]
        s = torch.cuda.Stream()
        before = atmm.overlap_stats()
        with torch.cuda.stream(s):
            for grp in groups:
                p.apply_group([work[x] for x, _ in grp], [work[y] for _, y in grp], [0] * len(grp), stream=s)
        s.synchronize()
        after = atmm.overlap_stats()
        early.append(after[1] - before[1])
        res.append(work)
    for u, v in zip(*res):
        assert torch.equal(u, v)
    # the second group is disjoint from the first; the third reads Y5 / Y6 / Y7 the second wrote (RAW)
    assert early[1] == 0 and early[0] <= 2


def _split_setup(atmm, oracle, seed=9):
    import torch

    reg = atmm.AdapterRegistry(2, D, D)
    rng = oracle.rng(seed)
    ranks = {0: 16, 1: 64, 2: 32}
    facs = {0: {}, 1: {}}
    for a, r in ranks.items():
        s = 1.0 / np.sqrt(np.float32(r))
        down = oracle.round_bf16(oracle.random_matrix(rng, 2 * D, r, -s, s).reshape(2, D, r))
        up = oracle.round_bf16(oracle.random_matrix(rng, 2 * r, D, -s, s).reshape(2, r, D))
        reg.put(a, down, up)
        for l in range(2):
            facs[l][a] = (down[l], up[l])
    assignment = np.repeat(np.asarray(sorted(ranks), np.int32), 128)
    assignment = assignment[np.random.default_rng(seed).permutation(assignment.size)]
    from conftest import path_table

    plan = atmm.BypassPlan(reg, assignment, path_table(atmm, assignment, ranks, D, D, "split"))
    ref_plan = atmm.BypassPlan(reg, assignment, path_table(atmm, assignment, ranks, D, D, "split"))
    ref_plan.set_overlap(False)
    assert {g["path_bf16"] for g in plan.describe()} == {"split"}
    n = assignment.size
    bufs = [torch.empty(n, D, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1) for _ in range(8)]
    return plan, ref_plan, bufs, assignment, facs


@pytest.mark.parametrize("steps,early_after_first", [
    ([(0, 1), (2, 3), (4, 5), (6, 7), (0, 3)], 4),   # independent: every shrink after the first runs early
    ([(0, 1), (1, 2), (2, 3), (3, 4)], 0),           # Y_i is X_i+1: the shrink must wait
    ([(0, 1), (2, 0), (0, 5)], 1),                   # WAR on X0 is harmless for the shrink; (0, 5) reads Y of (2, 0)
])
def test_split_shrink_early_same_bits(gpu, atmm, oracle, steps, early_after_first):
    """Split-path applies: the shrink computes under the preceding expand only
    when that expand's Y writes miss its X, with alternating scratch sets;
    results equal the full-dependency plan bit for bit, eager and captured."""
    import torch

    plan, ref_plan, bufs, _, _ = _split_setup(atmm, oracle)
    res = []
    for p in (plan, ref_plan):
        work = [b.clone() for b in bufs]
        s = torch.cuda.Stream()
        # (the first step's predecessor is whatever ran last on this -- pooled,
        # possibly reused -- stream: it may legitimately start early)
        with torch.cuda.stream(s):
            xi, yi = steps[0]
            p.apply(work[xi], work[yi], layer=0, stream=s)
            before = atmm.split_overlap_stats()
            for i, (xi, yi) in enumerate(steps[1:], start=1):
                p.apply(work[xi], work[yi], layer=i % 2, stream=s)
        s.synchronize()
        after = atmm.split_overlap_stats()
        if p is plan:
            assert after[0] - before[0] == len(steps) - 1
            assert after[1] - before[1] == early_after_first, (before, after)
        else:
            assert after[1] == before[1]
        res.append(work)
    for u, v in zip(*res):
        assert torch.equal(u, v)


def test_split_shrink_early_graph_fresh_inputs_oracle(gpu, atmm, oracle):
    """A captured graph of independent split applies (early shrinks, scratch
    sets alternating, odd step count so replays start on the other set)
    replayed twice, every output against the oracle."""
    import torch

    from conftest import tol_for

    plan, _, _, assignment, facs = _split_setup(atmm, oracle, seed=13)
    n = assignment.size
    steps = 5
    rng = oracle.rng(3)
    xs = [oracle.round_bf16(oracle.random_matrix(rng, n, D)) for _ in range(steps)]
    ys = [oracle.round_bf16(oracle.random_matrix(rng, n, D)) for _ in range(steps)]
    xt = [torch.from_numpy(x).to("cuda", torch.bfloat16) for x in xs]
    yt = [torch.from_numpy(y).to("cuda", torch.bfloat16) for y in ys]
    s = torch.cuda.Stream()
    warm = torch.empty_like(yt[0])
    with torch.cuda.stream(s):
        plan.apply(xt[0], warm, layer=0, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    before = atmm.split_overlap_stats()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        for i in range(steps):
            plan.apply(xt[i], yt[i], layer=i % 2, stream=s)
    after = atmm.split_overlap_stats()
    assert after[1] - before[1] == steps - 1
    for rep in range(2):
        for i in range(steps):
            yt[i].copy_(torch.from_numpy(ys[i]).to("cuda", torch.bfloat16))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        for i in range(steps):
            want = ys[i].astype(np.float64) + oracle.bypass_rows_f64(xs[i], assignment, facs[i % 2])
            got = yt[i].float().cpu().numpy()
            assert float(np.max(np.abs(got - want))) <= tol_for(want), (rep, i)
