"""Seeded random batches over the whole operator surface at once: any hidden
sizes (odd ones included), ranks 1..300 (chunked above 128), 1-12 adapters
with ragged segments, bf16 / fp32 Y, per-adapter and per-call scales, the
packaged tiling table choosing every launch -- against the oracle with the
north-star tolerance, plus bit-exact reruns and bit-exact routing."""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(48))
def test_random_batches_match_oracle(gpu, atmm, oracle, seed):
    import torch

    rng = np.random.default_rng(1000 + seed)
    d_in = int(rng.choice([64, 96, 200, 512, 777, 1024, 2048, 4096, 4100]))
    d_out = int(rng.choice([64, 130, 256, 515, 1024, 3000, 4096]))
    n_ad = int(rng.integers(1, 13))
    ids = sorted(int(v) for v in rng.choice(1000, size=n_ad, replace=False))
    rmax = min(d_in, d_out) - 1
    ranks = {a: int(min(rmax, rng.choice([1, 4, 8, 16, 24, 32, 64, 100, 128, 129, 200, 300]))) for a in ids}
    scales = {a: float(rng.choice([1.0, 0.5, -1.0, 0.3])) for a in ids}
    lens = [int(rng.integers(1, 300)) for _ in ids]
    reg = atmm.AdapterRegistry(2, d_in, d_out)
    facs = {}
    orng = oracle.rng(seed)
    for a in ids:
        r = ranks[a]
        s = 1.0 / np.sqrt(np.float32(r))
        down = oracle.round_bf16(oracle.random_matrix(orng, 2 * d_in, r, -s, s).reshape(2, d_in, r))
        up = oracle.round_bf16(oracle.random_matrix(orng, 2 * r, d_out, -s, s).reshape(2, r, d_out))
        reg.put(a, down, up, scales[a])
        facs[a] = (down[1] * np.float32(scales[a]), up[1])
    asg = np.concatenate([np.full(n, a, np.int32) for a, n in zip(ids, lens)])
    asg = asg[rng.permutation(asg.size)]
    n = asg.size
    x = oracle.round_bf16(oracle.random_matrix(orng, n, d_in))
    y0 = oracle.round_bf16(oracle.random_matrix(orng, n, d_out))
    call_scale = float(rng.choice([1.0, -0.5]))
    plan = atmm.BypassPlan(reg, asg)
    seg, off, rows = plan.routing()
    oseg, ooff, orows = oracle.plan_batch(asg)
    assert np.array_equal(seg, oseg) and np.array_equal(off, ooff) and np.array_equal(rows, orows)
    dt = torch.bfloat16 if seed % 2 == 0 else torch.float32
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    outs = []
    for _ in range(2):
        yt = torch.from_numpy(y0).to("cuda", dt)
        plan.apply(xt, yt, layer=1, scale=call_scale)
        outs.append(yt)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]), "reruns must be bit-identical"
    want = y0.astype(np.float64) + call_scale * oracle.bypass_rows_f64(x, asg, facs)
    got = outs[0].float().cpu().numpy()
    err = float(np.max(np.abs(got - want)))
    assert err <= tol_for(want), (seed, d_in, d_out, ranks, lens, str(dt), err)
