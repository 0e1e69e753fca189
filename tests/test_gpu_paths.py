"""GPU parity of each bypass kernel path against the oracle.

The launcher picks, per launch group, the all-to-all fused kernel (small,
latency-bound tiles), the split shrink + expand pair (large tiles) or the
general fused kernel.  A tiling-table entry's launch path (ATMM_PATH_*)
forces one where it applies, so every path
is checked on the same seeded inputs (bf16 and fp32 Y, several ranks, ragged
segments) against the restated reference, with the north-star tolerance
1e-2 * max(1, max|ref|) and bit-exact reruns (test_atmm.cpp:72-94).
"""
import numpy as np
import pytest

from conftest import path_table, tol_for

pytestmark = pytest.mark.gpu

CASES = [
    # d_in, d_out, {adapter: rank}, rows per segment (ragged, Zipf-like)
    (512, 512, {1: 16, 2: 32, 3: 64}, [200, 33, 7]),
    (1024, 768, {4: 8, 5: 16}, [129, 64]),
    (4096, 4096, {6: 16, 7: 64, 8: 32, 9: 16}, [300, 40, 17, 130]),
    (5120, 5120, {10: 64, 11: 64}, [128, 128]),
]


def _inputs(oracle, d_in, d_out, ranks, lens, seed=31):
    rng = oracle.rng(seed)
    facs = {}
    for a, r in ranks.items():
        s = 1.0 / np.sqrt(np.float32(r))
        facs[a] = (oracle.round_bf16(oracle.random_matrix(rng, d_in, r, -s, s)),
                   oracle.round_bf16(oracle.random_matrix(rng, r, d_out, -s, s)))
    ids = sorted(ranks)
    assignment = np.concatenate([np.full(n, ids[i], np.int32) for i, n in enumerate(lens)])
    assignment = assignment[np.random.default_rng(seed).permutation(assignment.size)]
    n = assignment.size
    x = oracle.round_bf16(oracle.random_matrix(rng, n, d_in))
    y0 = oracle.round_bf16(oracle.random_matrix(rng, n, d_out))
    return facs, assignment, x, y0


@pytest.mark.parametrize("path", ["a2a", "split", "fused", "stream"])
@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("ydt", ["bf16", "f32"])
def test_path_parity(gpu, atmm, oracle, path, case, ydt):
    import torch

    d_in, d_out, ranks, lens = CASES[case]
    facs, assignment, x, y0 = _inputs(oracle, d_in, d_out, ranks, lens)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    for a, (down, up) in facs.items():
        reg.put(a, down, up, scale=0.75)
    plan = atmm.BypassPlan(reg, assignment, path_table(atmm, assignment, ranks, d_in, d_out, path))
    want = y0.astype(np.float64) + 0.75 * 2.0 * oracle.bypass_rows_f64(x, assignment, facs)
    dt = torch.bfloat16 if ydt == "bf16" else torch.float32
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    outs = []
    for _ in range(2):
        yt = torch.from_numpy(y0).to("cuda", dt)
        plan.apply(xt, yt, layer=0, scale=2.0)
        torch.cuda.synchronize()
        outs.append(yt.float().cpu().numpy())
    assert np.max(np.abs(outs[0] - want)) <= tol_for(want)
    assert np.array_equal(outs[0], outs[1]), "reruns must be bit-identical"


def test_paths_agree_closely(gpu, atmm, oracle):
    """All three kernels compute the same rounding of the same sums up to
    one bf16 ulp of Y (they differ only in where mid is rounded)."""
    import torch

    d_in, d_out, ranks, lens = CASES[2]
    facs, assignment, x, y0 = _inputs(oracle, d_in, d_out, ranks, lens, seed=5)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    for a, (down, up) in facs.items():
        reg.put(a, down, up)
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    res = {}
    for path in ("a2a", "split", "fused"):
        plan = atmm.BypassPlan(reg, assignment, path_table(atmm, assignment, ranks, d_in, d_out, path))
        yt = torch.from_numpy(y0).to("cuda", torch.float32)
        plan.apply(xt, yt)
        torch.cuda.synchronize()
        res[path] = yt.cpu().numpy()
    want = y0.astype(np.float64) + oracle.bypass_rows_f64(x, assignment, facs)
    for path, got in res.items():
        assert np.max(np.abs(got - want)) <= tol_for(want), path
    assert np.max(np.abs(res["split"] - res["fused"])) <= tol_for(want)


def test_split_path_is_chosen_for_large_tiles(gpu, atmm, oracle):
    """The built-in heuristic's path choice (the packaged table may pick
    otherwise for shapes it profiled: it is checked in test_host.py)."""
    d_in, d_out, ranks, lens = CASES[3]
    facs, assignment, _, _ = _inputs(oracle, d_in, d_out, ranks, lens)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    for a, (down, up) in facs.items():
        reg.put(a, down, up)
    groups = atmm.BypassPlan(reg, assignment, use_default_table=False).describe()
    assert all(g["path_bf16"] == "split" for g in groups), groups
    small = np.repeat(np.asarray(sorted(ranks), np.int32), 16)
    groups = atmm.BypassPlan(reg, small, use_default_table=False).describe()
    assert all(g["path_bf16"] == "a2a" for g in groups), groups


@pytest.mark.parametrize("seed", range(8))
def test_random_shapes_all_paths(gpu, atmm, oracle, seed):
    """Random d_in / d_out (incl. not multiples of 8 or 64), ranks 1..128,
    ragged segments down to 1 row, bf16 and fp32 Y: every kernel path the
    launcher can take matches the oracle."""
    import torch

    rng = np.random.default_rng(1000 + seed)
    d_in = int(rng.integers(16, 1200))
    d_out = int(rng.choice([int(rng.integers(8, 1200)) // 8 * 8, int(rng.integers(9, 700))]))
    n_ad = int(rng.integers(1, 6))
    ranks = {int(a): int(rng.choice([1, 7, 16, 33, 64, 100, 128])) for a in rng.choice(50, n_ad, replace=False)}
    lens = [int(v) for v in rng.integers(1, 150, n_ad)]
    facs, assignment, x, y0 = _inputs(oracle, d_in, d_out, ranks, lens, seed=seed)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    for a, (down, up) in facs.items():
        reg.put(a, down, up)
    want_b = oracle.bypass_rows_f64(x, assignment, facs)
    # X rows must be 16-byte aligned (ldx % 8 == 0): pad the row stride, as a caller would
    ldx = (d_in + 7) // 8 * 8
    xpad = torch.zeros(x.shape[0], ldx, dtype=torch.bfloat16, device="cuda")
    xpad[:, :d_in] = torch.from_numpy(x).to("cuda", torch.bfloat16)
    xt = xpad[:, :d_in]
    for path in ("auto", "a2a", "split", "fused", "stream"):
        plan = atmm.BypassPlan(reg, assignment, path_table(atmm, assignment, ranks, d_in, d_out, path))
        for dt in (torch.bfloat16, torch.float32):
            yt = torch.from_numpy(y0).to("cuda", dt)
            plan.apply(xt, yt)
            torch.cuda.synchronize()
            want = y0.astype(np.float64) + want_b
            got = yt.float().cpu().numpy()
            assert np.max(np.abs(got - want)) <= tol_for(want), (path, dt, d_in, d_out, ranks, lens)


def test_large_batch_row_subset(gpu, atmm, oracle):
    """Maximum-size case: d = 8192, 64 rank-128 adapters,
    16384 ragged rows; rows are independent, so a row subset is checked
    against the oracle (and the whole output for finiteness)."""
    import torch

    d, n_ad = 8192, 64
    ranks = {a: 128 for a in range(n_ad)}
    rng = np.random.default_rng(77)
    lens = (rng.zipf(1.3, n_ad) % 900 + 1).astype(int)
    lens = (lens * (16384 / lens.sum())).astype(int) + 1
    reg = atmm.AdapterRegistry(1, d, d)
    orng = oracle.rng(5)
    facs = {}
    for a, r in ranks.items():
        s = 1.0 / np.sqrt(np.float32(r))
        facs[a] = (oracle.round_bf16(oracle.random_matrix(orng, d, r, -s, s)),
                   oracle.round_bf16(oracle.random_matrix(orng, r, d, -s, s)))
        reg.put(a, *facs[a])
    assignment = np.concatenate([np.full(int(m), a, np.int32) for a, m in zip(sorted(ranks), lens)])
    assignment = assignment[np.random.default_rng(3).permutation(assignment.size)]
    n = assignment.size
    x = torch.empty(n, d, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y0 = torch.empty(n, d, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y = y0.clone()
    plan = atmm.BypassPlan(reg, assignment)
    assert {g["path_bf16"] for g in plan.describe()} <= {"split", "a2a", "fused"}
    plan.apply(x, y)
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all()
    pick = np.random.default_rng(1).choice(n, 24, replace=False)
    xs = x[pick].float().cpu().numpy()
    want = y0[pick].float().cpu().numpy().astype(np.float64) + oracle.bypass_rows_f64(xs, assignment[pick], facs)
    got = y[pick].float().cpu().numpy()
    assert np.max(np.abs(got - want)) <= tol_for(want)


@pytest.mark.parametrize("path", ["a2a", "fused", "split", "stream"])
def test_x_ready_flag_same_results(gpu, atmm, oracle, path):
    """ATMM_PLAN_X_READY (X gathered before griddepcontrol.wait): K
    back-to-back applies on one stream over distinct (X, Y) buffers give the
    same bits as without the flag, and match the oracle."""
    import torch

    d_in, d_out, ranks, lens = CASES[2]
    facs, assignment, x, y0 = _inputs(oracle, d_in, d_out, ranks, lens, seed=5)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    for a, (down, up) in facs.items():
        reg.put(a, down, up)
    plan = atmm.BypassPlan(reg, assignment, path_table(atmm, assignment, ranks, d_in, d_out, path))
    K = 6
    rng = np.random.default_rng(3)
    xs = [torch.from_numpy(oracle.round_bf16(x * rng.uniform(0.5, 1.5))).to("cuda", torch.bfloat16) for _ in range(K)]
    ys0 = [torch.from_numpy(y0).to("cuda", torch.bfloat16) for _ in range(K)]
    runs = []
    for ready in (False, True):
        plan.set_x_ready(ready)
        ys = [y.clone() for y in ys0]
        torch.cuda.synchronize()
        for k in range(K):
            plan.apply(xs[k], ys[k], layer=0)
        torch.cuda.synchronize()
        runs.append([y.float().cpu().numpy() for y in ys])
    for k in range(K):
        assert np.array_equal(runs[0][k], runs[1][k]), k
    want = y0.astype(np.float64) + oracle.bypass_rows_f64(xs[K - 1].float().cpu().numpy(), assignment, facs)
    assert np.max(np.abs(runs[1][K - 1] - want)) <= tol_for(want)
    from paper_2411_00915_b200 import atmm as mod

    with pytest.raises(atmm.ConfigError):  # unknown flag bits
        mod._check(mod.lib.atmm_plan_set_flags(plan.handle, 8))
