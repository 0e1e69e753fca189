"""Back-to-back applies of one plan with DIFFERENT inputs each time, no
synchronisation in between, on every kernel path: consecutive launches then
overlap (programmatic dependent launch) and reuse the plan's scratch (mid,
partials, readiness counters, TMEM ring), so state left by one apply that the
next one reads too early shows up as a wrong result -- with identical inputs
the stale values would be the right ones and a rerun test could not see it.
Each apply is checked against the oracle."""
import numpy as np
import pytest

from conftest import path_table, tol_for

pytestmark = pytest.mark.gpu

CASES = [
    # (path, ranks, rows per adapter, d_in, d_out)
    ("a2a", {0: 16, 1: 8, 2: 32}, 24, 1024, 1024),
    ("a2a", {0: 32, 1: 16}, 32, 1024, 1024),
    ("split", {0: 16, 1: 64, 2: 32}, 128, 1024, 1024),
    ("split", {0: 128, 1: 8}, 200, 768, 1536),
    ("fused", {0: 16, 1: 48}, 70, 1024, 512),
    ("stream", {0: 32, 1: 16, 2: 64}, 96, 1024, 1024),
    ("auto", {0: 300, 1: 16, 2: 4}, 150, 1024, 1024),  # rank chunks: extra passes
]


@pytest.mark.parametrize("path,ranks,rows,d_in,d_out", CASES)
@pytest.mark.parametrize("ydt", ["bf16", "f32"])
@pytest.mark.parametrize("order", ["shuffled", "sorted"])  # sorted: tiles of consecutive rows (TMA boxes)
def test_back_to_back_fresh_inputs(gpu, atmm, oracle, path, ranks, rows, d_in, d_out, ydt, order):
    import torch

    reg = atmm.AdapterRegistry(2, d_in, d_out)
    facs = {0: {}, 1: {}}
    rng = oracle.rng(21)
    for a, r in ranks.items():
        s = 1.0 / np.sqrt(np.float32(r))
        down = oracle.round_bf16(oracle.random_matrix(rng, 2 * d_in, r, -s, s).reshape(2, d_in, r))
        up = oracle.round_bf16(oracle.random_matrix(rng, 2 * r, d_out, -s, s).reshape(2, r, d_out))
        reg.put(a, down, up)
        for l in range(2):
            facs[l][a] = (down[l], up[l])
    asg = np.repeat(np.asarray(sorted(ranks), np.int32), rows)
    if order == "shuffled":
        asg = asg[np.random.default_rng(4).permutation(asg.size)]
    n = asg.size
    table = path_table(atmm, asg, ranks, d_in, d_out, path) if path != "auto" and max(ranks.values()) <= 128 else None
    plan = atmm.BypassPlan(reg, asg, table)
    if table is not None:  # the forced path is the one that runs (bf16 Y; fp32 Y may take another)
        assert {g["path_bf16"] for g in plan.describe()} == {path}
    dt = torch.bfloat16 if ydt == "bf16" else torch.float32
    steps = 5
    xs = [oracle.round_bf16(oracle.random_matrix(rng, n, d_in)) for _ in range(steps)]
    ys = [oracle.round_bf16(oracle.random_matrix(rng, n, d_out)) for _ in range(steps)]
    xt = [torch.from_numpy(x).to("cuda", torch.bfloat16) for x in xs]
    yt = [torch.from_numpy(y).to("cuda", dt) for y in ys]
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(steps):
            plan.apply(xt[i], yt[i], layer=i % 2, stream=s)
    s.synchronize()
    for i in range(steps):
        want = ys[i].astype(np.float64) + oracle.bypass_rows_f64(xs[i], asg, facs[i % 2])
        got = yt[i].float().cpu().numpy()
        err = float(np.max(np.abs(got - want)))
        assert err <= tol_for(want), (path, ydt, i, err)
