"""GPU parity of the fused bypass against the oracle (restated reference).

Inputs are rounded to bf16 (RNE) before they reach either side, so the
oracle sees exactly the values the tensor cores multiply.  Tolerance is the
north-star bound 1e-2 * max(1, max|ref|) (BASELINE.json), bf16 in / fp32 acc.
Mirrors test_batch.cpp (plan routing, per-row oracle, zero adapter, flop
accounting, permutation equivariance, missing adapter).
"""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


def _factors(oracle, seed, L, d_in, d_out, r):
    rng = oracle.rng(seed)
    s = 1.0 / np.sqrt(np.float32(r))
    down = oracle.round_bf16(oracle.random_matrix(rng, L * d_in, r, -s, s).reshape(L, d_in, r))
    up = oracle.round_bf16(oracle.random_matrix(rng, L * r, d_out, -s, s).reshape(L, r, d_out))
    return down, up


def _setup(atmm, oracle, d_in, d_out, ranks, L=1, seed=900, scales=None):
    reg = atmm.AdapterRegistry(L, d_in, d_out)
    facs = {}
    for a, r in ranks.items():
        down, up = _factors(oracle, seed + a, L, d_in, d_out, r)
        reg.put(a, down, up, 1.0 if scales is None else scales[a])
        facs[a] = (down, up)
    return reg, facs


def _x(oracle, n, d, seed=77):
    return oracle.round_bf16(oracle.random_matrix(oracle.rng(seed), n, d))


@pytest.mark.parametrize(
    "d_in,d_out,ranks,n",
    [
        (48, 48, {1: 8, 2: 16, 5: 4}, 11),       # test_batch.cpp:63-80 shapes
        (64, 64, {1: 8, 2: 8}, 5),
        (256, 256, {3: 16, 9: 32, 4: 64}, 200),
        (512, 384, {1: 16, 2: 48}, 300),         # rectangular, rank not /16
        (1000, 520, {7: 24}, 129),               # d not multiple of 64/32, 2 tiles
    ],
)
def test_bypass_matches_oracle_small(gpu, atmm, oracle, d_in, d_out, ranks, n):
    reg, facs = _setup(atmm, oracle, d_in, d_out, ranks)
    ids = sorted(ranks)
    rng = np.random.default_rng(n)
    assignment = np.asarray([ids[i] for i in rng.integers(0, len(ids), n)], np.int32)
    x = _x(oracle, n, d_in)
    got = atmm.run_bypass(reg, x, assignment)
    want = oracle.bypass_rows_f64(x, assignment, {a: (f[0][0], f[1][0]) for a, f in facs.items()})
    assert got.shape == want.shape
    assert np.max(np.abs(got - want)) <= tol_for(want)
    if d_in == d_out:
        # the reference's own float algorithm (tiled fp32 ATMM) agrees too
        ref32 = oracle.run_bypass(x, assignment, {a: (f[0][0], f[1][0]) for a, f in facs.items()})
        assert np.max(np.abs(got - ref32)) <= tol_for(ref32)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_bypass_baseline_configs(gpu, atmm, oracle, name):
    from paper_2411_00915_b200.workloads import bypass_config

    w = bypass_config(name)
    reg, facs = _setup(atmm, oracle, w.d_in, w.d_out, w.ranks, seed=1000)
    x = _x(oracle, w.tokens, w.d_in, seed=7)
    got = atmm.run_bypass(reg, x, w.assignment)
    want = oracle.bypass_rows_f64(x, w.assignment, {a: (f[0][0], f[1][0]) for a, f in facs.items()})
    assert np.max(np.abs(got - want)) <= tol_for(want)
    # routing uploaded to HBM is bit-exact with plan_batch
    plan = atmm.BypassPlan(reg, w.assignment)
    seg, off, rows = plan.routing()
    oseg, ooff, orows = oracle.plan_batch(w.assignment)
    assert np.array_equal(seg, oseg) and np.array_equal(off, ooff) and np.array_equal(rows, orows)


def test_residual_fused_bf16_and_f32(gpu, atmm, oracle):
    import torch

    d, ranks, n = 512, {1: 16, 2: 32, 3: 64}, 257
    reg, facs = _setup(atmm, oracle, d, d, ranks)
    assignment = np.asarray([1 + (i * 7) % 3 for i in range(n)], np.int32)
    x = _x(oracle, n, d)
    y0 = oracle.round_bf16(oracle.random_matrix(oracle.rng(5), n, d))
    byp = oracle.bypass_rows_f64(x, assignment, {a: (f[0][0], f[1][0]) for a, f in facs.items()})
    plan = atmm.BypassPlan(reg, assignment)
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    for dtype in (torch.float32, torch.bfloat16):
        for scale in (1.0, -1.0, 0.5):
            yt = torch.from_numpy(y0).to("cuda", dtype)
            plan.apply(xt, yt, layer=0, scale=scale)
            torch.cuda.synchronize()
            got = yt.float().cpu().numpy()
            want = y0.astype(np.float64) + scale * byp
            assert np.max(np.abs(got - want)) <= tol_for(want), (dtype, scale)


def test_zero_adapter_exact_zero(gpu, atmm):
    reg = atmm.AdapterRegistry(1, 32, 32)
    reg.put(1, np.zeros((32, 4), np.float32), np.zeros((4, 32), np.float32))
    x = np.random.default_rng(1).uniform(-1, 1, (5, 32)).astype(np.float32)
    out = atmm.run_bypass(reg, x, [1] * 5)
    assert np.max(np.abs(out)) == 0.0


def test_missing_adapter_raises(gpu, atmm):
    reg = atmm.AdapterRegistry(1, 32, 32)
    x = np.zeros((2, 32), np.float32)
    with pytest.raises(atmm.UnknownAdapterError):
        atmm.run_bypass(reg, x, [1, 1])


def test_permutation_equivariance_exact(gpu, atmm, oracle):
    """test_batch.cpp:130-157: permuting rows permutes outputs bit-exactly."""
    d, n = 256, 90
    reg, _ = _setup(atmm, oracle, d, d, {1: 8, 2: 8, 3: 32})
    x = _x(oracle, n, d)
    assignment = np.asarray([(1, 2, 2, 1, 3)[i % 5] for i in range(n)], np.int32)
    base = atmm.run_bypass(reg, x, assignment)
    perm = oracle.seeded_shuffle(oracle.rng(44), np.arange(n)).astype(np.int64)
    permuted = atmm.run_bypass(reg, x[perm], assignment[perm])
    assert np.array_equal(permuted, base[perm])


def test_deterministic_reruns(gpu, atmm, oracle):
    """test_atmm.cpp:72-80: bit-identical across runs (no atomics)."""
    from paper_2411_00915_b200.workloads import bypass_config

    w = bypass_config("cfg3")
    reg, _ = _setup(atmm, oracle, w.d_in, w.d_out, w.ranks, seed=1000)
    x = _x(oracle, w.tokens, w.d_in, seed=7)
    a = atmm.run_bypass(reg, x, w.assignment)
    b = atmm.run_bypass(reg, x, w.assignment)
    assert np.array_equal(a, b)


def test_cluster_sizes_agree(gpu, atmm, oracle):
    """Every launch configuration (cluster 1..16, chunk 32..256, tile rows)
    computes the same bypass within tolerance."""
    d, n = 1024, 300
    ranks = {1: 16, 2: 64, 3: 8}
    reg, facs = _setup(atmm, oracle, d, d, ranks)
    x = _x(oracle, n, d)
    assignment = np.asarray([(1, 2, 3)[i % 3] for i in range(n)], np.int32)
    want = oracle.bypass_rows_f64(x, assignment, {a: (f[0][0], f[1][0]) for a, f in facs.items()})
    for sm100 in [(128, 1, 256, 0), (128, 2, 128, 2), (64, 3, 64, 3), (128, 5, 192, 0),
                  (32, 8, 256, 4), (128, 16, 64, 0), (128, 12, 128, 0)]:
        t = atmm.TilingTable()
        for m_bucket in range(32, 129, 32):
            for r in ranks.values():
                t.insert(m_bucket, d, r, (128, 128, 256, 128, 16, 64), 1, sm100=sm100)
        got = atmm.run_bypass(reg, x, assignment, table=t)
        assert np.max(np.abs(got - want)) <= tol_for(want), sm100


def test_multi_layer_registry(gpu, atmm, oracle):
    d, L = 128, 3
    reg, facs = _setup(atmm, oracle, d, d, {1: 16, 2: 32}, L=L)
    x = _x(oracle, 40, d)
    assignment = np.asarray([1, 2] * 20, np.int32)
    for layer in range(L):
        got = atmm.run_bypass(reg, x, assignment, layer=layer)
        want = oracle.bypass_rows_f64(x, assignment, {a: (f[0][layer], f[1][layer]) for a, f in facs.items()})
        assert np.max(np.abs(got - want)) <= tol_for(want)
    with pytest.raises(atmm.ConfigError):
        atmm.run_bypass(reg, x, assignment, layer=L)


def test_adapter_scale(gpu, atmm, oracle):
    d = 128
    reg, facs = _setup(atmm, oracle, d, d, {1: 16, 2: 16}, scales={1: 2.0, 2: -0.5})
    x = _x(oracle, 20, d)
    assignment = np.asarray([1, 2] * 10, np.int32)
    got = atmm.run_bypass(reg, x, assignment)
    want = oracle.bypass_rows_f64(x, assignment, {a: (f[0][0], f[1][0]) for a, f in facs.items()})
    want[assignment == 1] *= 2.0
    want[assignment == 2] *= -0.5
    assert np.max(np.abs(got - want)) <= tol_for(want)


def test_unaligned_y_rows(gpu, atmm, oracle):
    """Y rows that are not 16-byte aligned take the non-TMA epilogue path."""
    import torch

    d_in, d_out, n = 256, 777, 70
    reg, facs = _setup(atmm, oracle, d_in, d_out, {1: 16, 2: 32})
    assignment = np.asarray([1, 2] * 35, np.int32)
    x = _x(oracle, n, d_in)
    want = oracle.bypass_rows_f64(x, assignment, {a: (f[0][0], f[1][0]) for a, f in facs.items()})
    plan = atmm.BypassPlan(reg, assignment)
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    for dtype in (torch.float32, torch.bfloat16):
        yt = torch.zeros(n, d_out, dtype=dtype, device="cuda")
        plan.apply(xt, yt)
        torch.cuda.synchronize()
        assert np.max(np.abs(yt.float().cpu().numpy() - want)) <= tol_for(want), dtype


def test_pipelined_host_residual(gpu, atmm, oracle):
    """Serving path: micro-batches through pinned host buffers, H2D/kernel/D2H pipelined."""
    import torch

    d, n = 256, 64
    reg, facs = _setup(atmm, oracle, d, d, {1: 16, 2: 32}, L=2)
    assignment = np.asarray([1, 2] * (n // 2), np.int32)
    plan = atmm.BypassPlan(reg, assignment)
    xs, ys, wants, layers = [], [], [], []
    for i in range(5):
        x = oracle.round_bf16(oracle.random_matrix(oracle.rng(100 + i), n, d))
        y0 = oracle.round_bf16(oracle.random_matrix(oracle.rng(200 + i), n, d))
        layer = i % 2
        want = y0.astype(np.float64) + oracle.bypass_rows_f64(
            x, assignment, {a: (f[0][layer], f[1][layer]) for a, f in facs.items()})
        xt = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
        yt = torch.from_numpy(y0).to(torch.bfloat16).pin_memory()
        xs.append(xt.view(torch.int16).numpy().view(np.uint16))
        ys.append(yt.view(torch.int16).numpy().view(np.uint16))
        wants.append((want, yt))
        layers.append(layer)
    atmm.residual_host_bf16_pipelined(plan, xs, ys, layers)
    for want, yt in wants:
        got = yt.float().numpy()
        assert np.max(np.abs(got - want)) <= tol_for(want)


def test_grouped_apply_matches_single_calls(gpu, atmm, oracle):
    """atmm_bypass_apply_group: G independent (X, Y, layer) calls in one launch
    give bit-identical results to G single applies."""
    import torch

    L, d, n = 3, 1024, 96
    ranks = {1: 16, 2: 32, 3: 16}
    reg, facs = _setup(atmm, oracle, d, d, ranks, L=L)
    assignment = np.asarray([1 + (i * 5) % 3 for i in range(n)], np.int32)
    plan = atmm.BypassPlan(reg, assignment)
    xs = [torch.from_numpy(_x(oracle, n, d, seed=40 + c)).to("cuda", torch.bfloat16) for c in range(L)]
    y0 = [torch.from_numpy(_x(oracle, n, d, seed=50 + c)).to("cuda", torch.bfloat16) for c in range(L)]
    ya = [y.clone() for y in y0]
    yb = [y.clone() for y in y0]
    layers = [2, 0, 1]
    plan.apply_group(xs, ya, layers, scale=0.5)
    for c in range(L):
        plan.apply(xs[c], yb[c], layer=layers[c], scale=0.5)
    torch.cuda.synchronize()
    for c in range(L):
        assert torch.equal(ya[c], yb[c])
        want = y0[c].float().cpu().numpy().astype(np.float64) + 0.5 * oracle.bypass_rows_f64(
            xs[c].float().cpu().numpy(), assignment, {a: (f[0][layers[c]], f[1][layers[c]]) for a, f in facs.items()})
        assert np.max(np.abs(ya[c].float().cpu().numpy() - want)) <= tol_for(want)


def _split_path_case(atmm, oracle, L=2):
    """A plan whose bf16-Y groups take the split shrink + expand pair (tiles
    of > 32 rows), i.e. the path with per-stream scratch."""
    d, n = 1024, 640
    ranks = {1: 16, 2: 64, 3: 32}
    reg, facs = _setup(atmm, oracle, d, d, ranks, L=L)
    assignment = np.asarray([(1, 1, 2, 3, 2)[i % 5] for i in range(n)], np.int32)
    plan = atmm.BypassPlan(reg, assignment)
    assert "split" in {g["path_bf16"] for g in plan.describe()}
    return reg, facs, plan, assignment, d, n


def test_pipelined_host_split_path(gpu, atmm, oracle):
    """the pipelined host paths run applies of one plan on
    2-4 streams concurrently; split-path plans need per-stream scratch."""
    import torch

    reg, facs, plan, assignment, d, n = _split_path_case(atmm, oracle)
    xs, ys, outs, wants, wants_fresh, layers = [], [], [], [], [], []
    for i in range(8):
        x = oracle.round_bf16(oracle.random_matrix(oracle.rng(300 + i), n, d))
        y0 = oracle.round_bf16(oracle.random_matrix(oracle.rng(400 + i), n, d))
        layer = i % 2
        byp = oracle.bypass_rows_f64(x, assignment, {a: (f[0][layer], f[1][layer]) for a, f in facs.items()})
        xt = torch.from_numpy(x).to(torch.bfloat16).pin_memory()
        yt = torch.from_numpy(y0).to(torch.bfloat16).pin_memory()
        ot = torch.zeros(n, d, dtype=torch.bfloat16).pin_memory()
        xs.append(xt.view(torch.int16).numpy().view(np.uint16))
        ys.append(yt.view(torch.int16).numpy().view(np.uint16))
        outs.append(ot.view(torch.int16).numpy().view(np.uint16))
        wants.append((y0.astype(np.float64) + byp, yt))
        wants_fresh.append((byp, ot))
        layers.append(layer)
    atmm.residual_host_bf16_pipelined(plan, xs, ys, layers)
    for want, yt in wants:
        assert np.max(np.abs(yt.float().numpy() - want)) <= tol_for(want)
    atmm.run_bypass_host_bf16_pipelined(plan, xs, outs, layers)
    for want, ot in wants_fresh:
        assert np.max(np.abs(ot.float().numpy() - want)) <= tol_for(want)


def test_split_plan_concurrent_streams_bit_identical(gpu, atmm, oracle):
    """Applies of one split-path plan on several streams at once give the
    same bits as the serialized applies."""
    import torch

    reg, facs, plan, assignment, d, n = _split_path_case(atmm, oracle)
    S = 4
    xs = [torch.from_numpy(_x(oracle, n, d, seed=60 + c)).to("cuda", torch.bfloat16) for c in range(S)]
    y0 = [torch.from_numpy(_x(oracle, n, d, seed=70 + c)).to("cuda", torch.bfloat16) for c in range(S)]
    K = 3  # each stream accumulates K applies into its own Y
    ser = [y.clone() for y in y0]
    for c in range(S):
        for _ in range(K):
            plan.apply(xs[c], ser[c], layer=c % 2)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(S)]
    for rep in range(3):
        par = [y.clone() for y in y0]
        torch.cuda.synchronize()
        for _ in range(K):  # interleaved issue: every stream has work in flight
            for c in range(S):
                plan.apply(xs[c], par[c], layer=c % 2, stream=streams[c])
        torch.cuda.synchronize()
        for c in range(S):
            assert torch.equal(par[c], ser[c]), (rep, c)
