"""GPU parity of each bypass kernel path against the oracle.

The launcher picks, per launch group, the all-to-all fused kernel (small,
latency-bound tiles), the split shrink + expand pair (large tiles) or the
general fused kernel.  ATMM_PATH forces one where it applies, so every path
is checked on the same seeded inputs (bf16 and fp32 Y, several ranks, ragged
segments) against the restated reference, with the north-star tolerance
1e-2 * max(1, max|ref|) and bit-exact reruns (test_atmm.cpp:72-94).
"""
import numpy as np
import pytest

from conftest import tol_for

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


@pytest.mark.parametrize("path", ["a2a", "split", "fused"])
@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("ydt", ["bf16", "f32"])
def test_path_parity(gpu, atmm, oracle, monkeypatch, path, case, ydt):
    import torch

    monkeypatch.setenv("ATMM_PATH", path)
    d_in, d_out, ranks, lens = CASES[case]
    facs, assignment, x, y0 = _inputs(oracle, d_in, d_out, ranks, lens)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    for a, (down, up) in facs.items():
        reg.put(a, down, up, scale=0.75)
    plan = atmm.BypassPlan(reg, assignment)
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


def test_paths_agree_closely(gpu, atmm, oracle, monkeypatch):
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
        monkeypatch.setenv("ATMM_PATH", path)
        plan = atmm.BypassPlan(reg, assignment)
        yt = torch.from_numpy(y0).to("cuda", torch.float32)
        plan.apply(xt, yt)
        torch.cuda.synchronize()
        res[path] = yt.cpu().numpy()
    want = y0.astype(np.float64) + oracle.bypass_rows_f64(x, assignment, facs)
    for path, got in res.items():
        assert np.max(np.abs(got - want)) <= tol_for(want), path
    assert np.max(np.abs(res["split"] - res["fused"])) <= tol_for(want)


def test_split_path_is_chosen_for_large_tiles(gpu, atmm, oracle, monkeypatch):
    monkeypatch.delenv("ATMM_PATH", raising=False)
    d_in, d_out, ranks, lens = CASES[3]
    facs, assignment, _, _ = _inputs(oracle, d_in, d_out, ranks, lens)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    for a, (down, up) in facs.items():
        reg.put(a, down, up)
    groups = atmm.BypassPlan(reg, assignment).describe()
    assert all(g["path_bf16"] == "split" for g in groups), groups
    small = np.repeat(np.asarray(sorted(ranks), np.int32), 16)
    groups = atmm.BypassPlan(reg, small).describe()
    assert all(g["path_bf16"] == "a2a" for g in groups), groups
