"""GPU parity of the fused mixture (deLoRA) bypass against the oracle.

forward_mixture (model.hpp:252-328): rows of the merged adapter get no
bypass (they ride the merged weights); every guest row gets its own
adapter's bypass minus the merged adapter's (the subtraction branch), added
into Y.  Our MixturePlan does both in ONE fused launch through a combined
slot (rank concatenation, sign folded into up).  Tolerance 1e-2 max(1, |ref|).
"""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


def _reg(atmm, oracle, d_in, d_out, ranks, seed=4):
    rng = oracle.rng(seed)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    facs = {}
    for a, r in ranks.items():
        s = 1.0 / np.sqrt(np.float32(r))
        f = (oracle.round_bf16(oracle.random_matrix(rng, d_in, r, -s, s)),
             oracle.round_bf16(oracle.random_matrix(rng, r, d_out, -s, s)))
        reg.put(a, *f)
        facs[a] = f
    return reg, facs


@pytest.mark.parametrize("d,ranks,merged,n", [
    (512, {1: 16, 2: 32, 3: 64}, 3, 300),
    (4096, {1: 16, 2: 16, 5: 64, 7: 8}, 1, 512),
    (1024, {4: 48, 9: 16}, 9, 77),
])
@pytest.mark.parametrize("ydt", ["bf16", "f32"])
def test_mixture_matches_oracle(gpu, atmm, oracle, d, ranks, merged, n, ydt):
    import torch

    reg, facs = _reg(atmm, oracle, d, d, ranks)
    ids = sorted(ranks)
    assignment = np.asarray([ids[i] for i in np.random.default_rng(n).integers(0, len(ids), n)], np.int32)
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(11), n, d))
    y0 = oracle.round_bf16(oracle.random_matrix(oracle.rng(12), n, d))
    guest = assignment != merged
    own = oracle.bypass_rows_f64(x, assignment, facs)
    cancel = oracle.bypass_rows_f64(x, np.full(n, merged, np.int32), facs)
    want = y0.astype(np.float64) + np.where(guest[:, None], own - cancel, 0.0)
    mp = atmm.MixturePlan(reg, assignment, merged)
    dt = torch.bfloat16 if ydt == "bf16" else torch.float32
    yt = torch.from_numpy(y0).to("cuda", dt)
    mp.apply(torch.from_numpy(x).to("cuda", torch.bfloat16), yt)
    torch.cuda.synchronize()
    got = yt.float().cpu().numpy()
    assert np.max(np.abs(got - want)) <= tol_for(want)
    # merged rows are untouched, bit for bit
    assert np.array_equal(got[~guest], y0[~guest].astype(np.float32) if ydt == "f32" else
                          torch.from_numpy(y0[~guest]).to(torch.bfloat16).float().numpy())


def test_mixture_errors_and_edge_cases(gpu, atmm, oracle):
    import torch

    reg, facs = _reg(atmm, oracle, 256, 256, {1: 16, 2: 16})
    with pytest.raises(atmm.ModeError):
        atmm.MixturePlan(reg, [1, 2], 5)
    with pytest.raises(atmm.UnknownAdapterError):
        atmm.MixturePlan(reg, [1, 8], 2)
    # every row on the merged adapter: no bypass at all
    y = torch.ones(4, 256, device="cuda")
    atmm.MixturePlan(reg, [2, 2, 2, 2], 2).apply(torch.ones(4, 256, device="cuda", dtype=torch.bfloat16), y)
    torch.cuda.synchronize()
    assert bool((y == 1).all())
    # combined rank above 128: those guests take the two-pass form (own, then
    # cancel with scale -1), same values within bf16 rounding
    rng = np.random.default_rng(8)
    d3 = rng.uniform(-0.1, 0.1, (256, 120)).astype(np.float32)
    u3 = rng.uniform(-0.1, 0.1, (120, 256)).astype(np.float32)
    reg.put(3, d3, u3)
    mp = atmm.MixturePlan(reg, [1, 3, 3], 3)
    assert mp.own is not None and list(mp.two_pass_rows) == [0]
    xm = torch.ones(3, 256, device="cuda", dtype=torch.bfloat16)
    ym = torch.zeros(3, 256, device="cuda")
    mp.apply(xm, ym)
    torch.cuda.synchronize()
    f1, f3 = facs[1], (oracle.round_bf16(d3), oracle.round_bf16(u3))
    ones = np.ones((1, 256))
    want = ones @ f1[0].astype(np.float64) @ f1[1] - ones @ f3[0].astype(np.float64) @ f3[1]
    assert np.max(np.abs(ym[0:1].cpu().numpy() - want)) <= tol_for(want)
    assert bool((ym[1:] == 0).all())
    with pytest.raises(atmm.ConfigError):
        atmm.LayerForward(mp)


def test_mixture_equals_two_pass_composition(gpu, atmm, oracle):
    """One fused launch vs the two-pass form (own plan, then the cancel
    plan with scale -1): same values within bf16 rounding of Y."""
    import torch

    d, n, merged = 1024, 256, 2
    reg, facs = _reg(atmm, oracle, d, d, {1: 16, 2: 32, 3: 64})
    assignment = np.asarray([1 + (i % 3) for i in range(n)], np.int32)
    x = torch.from_numpy(oracle.round_bf16(oracle.random_matrix(oracle.rng(3), n, d))).to("cuda", torch.bfloat16)
    y1 = torch.zeros(n, d, device="cuda")
    atmm.MixturePlan(reg, assignment, merged).apply(x, y1)
    guest = np.nonzero(assignment != merged)[0].astype(np.int32)
    y2 = torch.zeros(n, d, device="cuda")
    atmm.BypassPlan(reg, assignment[guest], rows=guest, n_rows=n).apply(x, y2)
    atmm.BypassPlan(reg, np.full(guest.size, merged, np.int32), rows=guest, n_rows=n).apply(x, y2, scale=-1.0)
    torch.cuda.synchronize()
    a, b = y1.cpu().numpy(), y2.cpu().numpy()
    assert np.max(np.abs(a - b)) <= 1e-2 * max(1.0, float(np.max(np.abs(b))))
