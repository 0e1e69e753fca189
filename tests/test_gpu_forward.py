"""GPU parity of the layer forward (model.hpp:192-328) against the oracle.

LayerForward runs cur <- tanh(cur @ W_l + bypass_l(cur)) for every layer:
the batched-LoRA bypass rides the base GEMM as extra K blocks of the same
tensor-core accumulator (forward_kernels.cu).  Checked against
orc_forward_f64 (the oracle restatement, itself pinned to the reference's
forward_* in tests/test_oracle.py) with bf16-rounded activations between
layers, at the north-star tolerance 1e-2 * max(1, max|ref|), plus the
reference's own golden forward outputs, bit-identical reruns and the
mode-equivalence property of verify.hpp:63-100.
"""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


def _model(atmm, oracle, L, d, ranks, seed=3):
    """bf16-exact W [L][d][d] (U(+-1/sqrt d), model.hpp:44-47) and adapters
    (U(+-1/sqrt r), adapter.hpp:60-64) in a registry."""
    w = oracle.round_bf16(oracle.model_random(seed, L, d))
    reg = atmm.AdapterRegistry(L, d)
    facs = {}
    for a, r in ranks.items():
        dn, up = oracle.adapter_random(1000 * seed + a, L, d, r)
        dn, up = oracle.round_bf16(dn), oracle.round_bf16(up)
        reg.put(a, dn, up)
        facs[a] = (dn, up)
    return w, reg, facs


def _dev(a, dtype=None):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype or torch.bfloat16)


def _assignment(ranks, lens, seed):
    ids = sorted(ranks)
    a = np.concatenate([np.full(n, ids[i % len(ids)], np.int32) for i, n in enumerate(lens)])
    return a[np.random.default_rng(seed).permutation(a.size)]


CASES = [
    # L, d, {adapter: rank}, rows per segment (ragged)
    (3, 256, {1: 16, 2: 32, 3: 64, 4: 128}, [60, 33, 7, 130]),
    (2, 512, {5: 8, 6: 16}, [129, 64]),
    (1, 1024, {7: 64, 8: 48, 9: 16}, [300, 41, 2]),
    (2, 128, {1: 96}, [5]),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_forward_unmerged_parity(gpu, atmm, oracle, case):
    import torch

    L, d, ranks, lens = CASES[case]
    w, reg, facs = _model(atmm, oracle, L, d, ranks, seed=case + 1)
    a = _assignment(ranks, lens, case)
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(7 + case), a.size, d))
    want = oracle.forward_f64(x, w, "unmerged", a, facs)
    fw = atmm.LayerForward(atmm.BypassPlan(reg, a))
    wt, xt = _dev(w), _dev(x)
    outs = []
    for _ in range(2):
        outs.append(fw.run(wt, xt).float().cpu().numpy())
        torch.cuda.synchronize()
    assert np.max(np.abs(outs[0] - want)) <= tol_for(want)
    assert np.array_equal(outs[0], outs[1]), "reruns must be bit-identical"


@pytest.mark.parametrize("d,n,L", [(256, 200, 3), (1024, 64, 2), (136, 7, 1)])
def test_forward_merged_parity(gpu, atmm, oracle, d, n, L):
    w = oracle.round_bf16(oracle.model_random(d + n, L, d))
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(n), n, d))
    want = oracle.forward_f64(x, w, "merged")
    got = atmm.forward_merged(_dev(w), _dev(x)).float().cpu().numpy()
    assert np.max(np.abs(got - want)) <= tol_for(want)


@pytest.mark.parametrize("merged", [2, 4])
def test_forward_mixture_parity_and_mode_equivalence(gpu, atmm, oracle, merged):
    """forward_mixture over merged weights matches the oracle; rows of the
    merged adapter equal forward_merged bit for bit (they get no bypass and
    the same GEMM), the rest match forward_unmerged within tolerance
    (verify.hpp:89-100)."""
    L, d = 3, 256
    ranks = {1: 16, 2: 32, 4: 64}
    w, reg, facs = _model(atmm, oracle, L, d, ranks, seed=9)
    a = _assignment(ranks, [70, 50, 90], 4)
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(21), a.size, d))
    wm = oracle.round_bf16(oracle.merge(w, facs[merged][0], facs[merged][1], +1))
    want = oracle.forward_f64(x, wm, "mixture", a, facs, merged_id=merged)
    got = atmm.forward_mixture(_dev(wm), _dev(x), a, reg, merged).float().cpu().numpy()
    assert np.max(np.abs(got - want)) <= tol_for(want)
    merged_rows = atmm.forward_merged(_dev(wm), _dev(x)).float().cpu().numpy()
    host = a == merged
    assert np.array_equal(got[host], merged_rows[host])
    # guest rows vs the unmerged forward: two computations, each within tol of
    # its own exact value (the merged W carries its own bf16 rounding of dW)
    unmerged = oracle.forward_f64(x, w, "unmerged", a, facs)
    assert np.max(np.abs(got[~host] - unmerged[~host])) <= 2 * tol_for(unmerged)


def test_forward_reference_golden(gpu, atmm, oracle):
    """The reference's own forward_unmerged / forward_mixture / forward_merged
    outputs (tests/golden, verify.hpp:63-100 setting) reproduced on device
    from bf16-rounded inputs."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))
    L, d = g["fwd_w"].shape[0], g["fwd_w"].shape[1]
    reg = atmm.AdapterRegistry(L, d)
    for a in (1, 2):
        reg.put(a, oracle.round_bf16(g[f"fwd_down_{a}"]), oracle.round_bf16(g[f"fwd_up_{a}"]))
    x = _dev(oracle.round_bf16(g["fwd_x"]))
    asg = g["fwd_assignment"]
    got = atmm.forward_unmerged(_dev(oracle.round_bf16(g["fwd_w"])), x, asg, reg).float().cpu().numpy()
    assert np.max(np.abs(got - g["fwd_unmerged"])) <= tol_for(g["fwd_unmerged"])
    wm = _dev(oracle.round_bf16(g["fwd_w_merged"]))
    got = atmm.forward_mixture(wm, x, asg, reg, 1).float().cpu().numpy()
    assert np.max(np.abs(got - g["fwd_mixture"])) <= tol_for(g["fwd_mixture"])
    got = atmm.forward_merged(wm, x).float().cpu().numpy()
    assert np.max(np.abs(got - g["fwd_merged"])) <= tol_for(g["fwd_merged"])


@pytest.mark.parametrize("seed", range(6))
def test_forward_random_shapes(gpu, atmm, oracle, seed):
    """Random hidden sizes (multiples of 8, not of 64), ragged segments down
    to one row, ranks 1..128, both GEMM tile widths and shrink K splits."""
    rng = np.random.default_rng(500 + seed)
    d = int(rng.integers(2, 80)) * 8
    L = int(rng.integers(1, 4))
    n_ad = int(rng.integers(1, 7))
    ranks = {int(a): int(rng.choice([1, 7, 16, 33, 64, 100, 128])) for a in rng.choice(40, n_ad, replace=False)}
    lens = [int(v) for v in rng.integers(1, 90, n_ad)]
    w, reg, facs = _model(atmm, oracle, L, d, ranks, seed=seed + 20)
    a = _assignment(ranks, lens, seed)
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(seed), a.size, d))
    want = oracle.forward_f64(x, w, "unmerged", a, facs)
    for bn, ks, pair, kz in [("128", None, "1", "1"), ("256", "1", "1", "1"), ("256", "4", "0", "1"),
                             ("128", "2", "0", "1"), ("128", "2", "0", "4"), ("128", None, "0", "2")]:
        opts = {"bn": int(bn), "pair": int(pair), "kz": int(kz), "ks": int(ks or 0)}
        got = atmm.LayerForward(atmm.BypassPlan(reg, a), opts=opts).run(_dev(w), _dev(x)).float().cpu().numpy()
        assert np.max(np.abs(got - want)) <= tol_for(want), (bn, ks, pair, kz, d, L, ranks, lens)


def test_forward_large_rows_subset(gpu, atmm, oracle):
    """cfg2's shape (d = 4096, 512 tokens, 16 rank-16 adapters), two layers:
    rows are independent, so a row subset checks the full-size launch."""
    L, d = 2, 4096
    ranks = {i: 16 for i in range(16)}
    w, reg, facs = _model(atmm, oracle, L, d, ranks, seed=2)
    a = _assignment(ranks, [32] * 16, 1)
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(3), a.size, d))
    got = atmm.LayerForward(atmm.BypassPlan(reg, a)).run(_dev(w), _dev(x)).float().cpu().numpy()
    pick = np.random.default_rng(0).choice(a.size, 12, replace=False)
    want = oracle.forward_f64(x[pick], w, "unmerged", a[pick], facs)
    assert np.max(np.abs(got[pick] - want)) <= tol_for(want)


def test_forward_errors_and_edges(gpu, atmm, oracle):
    import torch

    L, d = 2, 128
    w, reg, facs = _model(atmm, oracle, L, d, {1: 16}, seed=5)
    a = np.asarray([1, 1, 1], np.int32)
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(1), 3, d))
    fw = atmm.LayerForward(atmm.BypassPlan(reg, a))
    # zero layers copies X
    out = fw.run(_dev(w), _dev(x), num_layers=0)
    assert np.array_equal(out.float().cpu().numpy(), x)
    with pytest.raises(atmm.ShapeError):
        fw.run(_dev(w), _dev(x), num_layers=L + 1)
    with pytest.raises(atmm.ShapeError):
        fw.run(_dev(w[:, :64, :64]), _dev(x))
    # replacing an adapter makes the forward stale
    reg.put(1, *facs[1])
    with pytest.raises(atmm.ConfigError):
        fw.run(_dev(w), _dev(x))
    with pytest.raises(atmm.ShapeError):
        atmm.LayerForward(None, n=4, hidden_dim=100)
    torch.cuda.synchronize()


GEMM_CASES = [(1, 64, 8), (7, 104, 136), (130, 256, 512), (300, 1000, 264), (257, 72, 1024), (512, 4096, 4096),
              (257, 192, 512), (384, 576, 264)]  # odd counts of 64-wide K blocks under 128-deep stages


@pytest.mark.parametrize("m,k,n", GEMM_CASES)
@pytest.mark.parametrize("out", ["bf16", "f32"])
def test_gemm_parity(gpu, atmm, oracle, m, k, n, out):
    """atmm_gemm (the base GEMM of model.hpp:238, atmm_multiply_into with a
    dense operand) against an fp64 product of the same bf16 inputs, over the
    1-SM, split-K and 2-SM tile paths; reruns bit-identical."""
    import torch

    rng = np.random.default_rng(m * 7 + k + n)
    a = oracle.round_bf16(rng.uniform(-1, 1, (m, k)))
    b = oracle.round_bf16(rng.uniform(-1, 1, (k, n)) / np.sqrt(k))
    want = a @ b
    dt = torch.float32 if out == "f32" else torch.bfloat16
    for opts in [{"pair": 1, "kz": 1}, {"pair": 0, "kz": 1}, {"pair": 0, "kz": 2}, {"pair": 0, "kz": 4},
                 {"pair": 0, "bn": 256}, {"pair": 1, "bn": 128}, {"pair": 0, "stages": 2}, None]:
        at, bt = _dev(a), _dev(b)
        got = atmm.gemm(at, bt, out_dtype=dt, opts=opts)
        again = atmm.gemm(at, bt, out_dtype=dt, opts=opts)
        torch.cuda.synchronize()
        g = got.float().cpu().numpy()
        assert np.max(np.abs(g - want)) <= tol_for(want), opts
        assert torch.equal(got, again)


def test_gemm_strides_and_edges(gpu, atmm, oracle):
    import torch

    rng = np.random.default_rng(1)
    a = oracle.round_bf16(rng.uniform(-1, 1, (70, 96)))
    b = oracle.round_bf16(rng.uniform(-1, 1, (96, 40)))
    abig = torch.zeros(70, 128, device="cuda", dtype=torch.bfloat16)
    abig[:, :96] = _dev(a)
    bbig = torch.zeros(96, 64, device="cuda", dtype=torch.bfloat16)
    bbig[:, :40] = _dev(b)
    cbig = torch.full((70, 48), 7.0, device="cuda")
    atmm.gemm(abig[:, :96], bbig[:, :40], out=cbig[:, :40])
    got = cbig.cpu().numpy()
    assert np.max(np.abs(got[:, :40] - a @ b)) <= tol_for(a @ b)
    assert np.all(got[:, 40:] == 7.0), "columns past n must not be written"
    # k = 0 zeroes C; m = 0 is a no-op
    c = torch.full((5, 8), 3.0, device="cuda")
    atmm.gemm(torch.empty(5, 0, device="cuda", dtype=torch.bfloat16),
              torch.empty(0, 8, device="cuda", dtype=torch.bfloat16), out=c)
    assert torch.count_nonzero(c) == 0
    atmm.gemm(torch.empty(0, 16, device="cuda", dtype=torch.bfloat16), _dev(b[:16, :8]))
    with pytest.raises(atmm.ShapeError):
        atmm.gemm(_dev(a), _dev(b[:, :36]))          # n not a multiple of 8
    with pytest.raises(atmm.ShapeError):
        atmm.gemm(_dev(a), _dev(b[:64]))             # shapes do not chain
    torch.cuda.synchronize()


@pytest.mark.parametrize("mc", ["2", "4"])
@pytest.mark.parametrize("m,k,n", [(1, 64, 512), (130, 1000, 1024), (300, 4096, 2048)])
def test_gemm_a_multicast(gpu, atmm, oracle, mc, m, k, n):
    """The 1-SM GEMM with A multicast over clusters of mc N tiles."""
    import torch

    opts = {"pair": 0, "bn": 128, "mc": int(mc)}
    rng = np.random.default_rng(m + k + n)
    a = oracle.round_bf16(rng.uniform(-1, 1, (m, k)))
    b = oracle.round_bf16(rng.uniform(-1, 1, (k, n)) / np.sqrt(k))
    want = a @ b
    at, bt = _dev(a), _dev(b)
    got = atmm.gemm(at, bt, out_dtype=torch.float32, opts=opts)
    again = atmm.gemm(at, bt, out_dtype=torch.float32, opts=opts)
    torch.cuda.synchronize()
    assert np.max(np.abs(got.cpu().numpy() - want)) <= tol_for(want)
    assert torch.equal(got, again)


def test_gemm_options_validated(gpu, atmm):
    import torch

    a = torch.zeros(8, 64, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(64, 8, device="cuda", dtype=torch.bfloat16)
    for bad in ({"bn": 192}, {"kz": 3}, {"pair": 2}, {"stages": 1}, {"mc": 3}):
        with pytest.raises(atmm.ConfigError):
            atmm.gemm(a, b, opts=bad)
    with pytest.raises(atmm.ConfigError):
        atmm.gemm(a, b, opts={"tile": 1})
