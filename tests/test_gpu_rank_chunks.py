"""Adapters above rank 128 (the reference accepts any rank below the hidden
size, adapter.hpp:30-31): stored as 128-rank chunk slots, applied as extra
row-mapped passes over the same X / Y (device.cu atmm_plan::passes), merged
and delta_w'd chunk by chunk.  Checked against the oracle with the
north-star tolerance; routing stays bit-exact (plan_batch, batch.hpp:28-42).
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


@pytest.mark.parametrize("ydt", ["bf16", "f32"])
@pytest.mark.parametrize("d_in,d_out,ranks,lens", [
    (1024, 1024, {1: 200, 2: 16, 3: 300}, [70, 33, 150]),        # 2- and 3-chunk adapters beside a small one
    (768, 512, {4: 129, 5: 256}, [5, 260]),                       # chunk boundary + 1, exact multiple
    (4096, 4096, {6: 320, 7: 64}, [32, 32]),                      # a2a-sized tiles
])
def test_chunked_rank_bypass_matches_oracle(gpu, atmm, oracle, ydt, d_in, d_out, ranks, lens):
    import torch

    L = 2
    reg = atmm.AdapterRegistry(L, d_in, d_out)
    facs = {}
    for a, r in ranks.items():
        down, up = _factors(oracle, 50 + a, L, d_in, d_out, r)
        reg.put(a, down, up)
        facs[a] = (down[1], up[1])
        assert reg.rank(a) == r
    ids = sorted(ranks)
    asg = np.concatenate([np.full(n, ids[i], np.int32) for i, n in enumerate(lens)])
    asg = asg[np.random.default_rng(3).permutation(asg.size)]
    n = asg.size
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(9), n, d_in))
    y0 = oracle.round_bf16(oracle.random_matrix(oracle.rng(10), n, d_out))
    plan = atmm.BypassPlan(reg, asg)
    passes = {g["pass"] for g in plan.describe()}
    assert passes == set(range(max((r + 127) // 128 for r in ranks.values()))), plan.describe()
    seg, off, rows = plan.routing()
    oseg, ooff, orows = oracle.plan_batch(asg)
    assert np.array_equal(seg, oseg) and np.array_equal(off, ooff) and np.array_equal(rows, orows)
    dt = torch.bfloat16 if ydt == "bf16" else torch.float32
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    yt = torch.from_numpy(y0).to("cuda", dt)
    plan.apply(xt, yt, layer=1)
    again = torch.from_numpy(y0).to("cuda", dt)
    plan.apply(xt, again, layer=1)
    torch.cuda.synchronize()
    assert torch.equal(yt, again), "reruns must be bit-identical"
    want = y0.astype(np.float64) + oracle.bypass_rows_f64(x, asg, facs)
    got = yt.float().cpu().numpy()
    assert np.max(np.abs(got - want)) <= tol_for(want)


def test_chunked_rank_delta_w_and_merge_round_trip(gpu, atmm, oracle):
    import torch

    d_in, d_out, r = 640, 896, 300
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    down, up = _factors(oracle, 77, 1, d_in, d_out, r)
    reg.put(11, down, up, 0.5)
    want = 0.5 * (down[0].astype(np.float64) @ up[0].astype(np.float64))
    dw = atmm.delta_w(reg, 11)
    assert np.max(np.abs(dw - want)) <= 1e-4 * max(1.0, float(np.abs(want).max()))
    w0 = oracle.random_matrix(oracle.rng(4), d_in, d_out)
    w = torch.from_numpy(w0).cuda()
    atmm.merge_into(reg, 11, 0, w)
    torch.cuda.synchronize()
    assert np.max(np.abs(w.cpu().numpy() - (w0 + want))) <= tol_for(w0 + want)
    atmm.merge_into(reg, 11, 0, w, sign=-1.0)
    torch.cuda.synchronize()
    assert np.max(np.abs(w.cpu().numpy() - w0)) <= 1e-4 * max(1.0, float(np.abs(w0).max()))


def test_chunked_rank_registry_lifecycle_and_limits(gpu, atmm, oracle):
    d = 512
    reg = atmm.AdapterRegistry(1, d, d)
    down, up = _factors(oracle, 5, 1, d, d, 260)
    reg.put(1, down, up)
    b3 = reg.nbytes()
    small_d, small_u = _factors(oracle, 6, 1, d, d, 16)
    reg.put(1, small_d, small_u)  # replacing a chunked adapter frees its extra chunks
    assert reg.rank(1) == 16 and reg.nbytes() < b3
    reg.put(1, down, up)
    assert reg.rank(1) == 260
    reg.remove(1)
    assert 1 not in reg and reg.nbytes() == 0
    big_d, big_u = _factors(oracle, 7, 1, d, d, d)  # rank == hidden size: the reference's ConfigError
    with pytest.raises(atmm.ConfigError):
        reg.put(2, big_d, big_u)
    reg.put(3, down, up)
    plan = atmm.BypassPlan(reg, np.full(40, 3, np.int32))
    with pytest.raises(atmm.ConfigError):
        atmm.LayerForward(plan)


def test_chunk_passes_keep_their_order(gpu, atmm, oracle):
    """The passes update the same Y rows: the launcher never starts one under
    the other (same bits as a plan with ATMM_PLAN_NO_OVERLAP)."""
    import torch

    d = 1024
    reg = atmm.AdapterRegistry(1, d, d)
    for a in range(4):
        down, up = _factors(oracle, 90 + a, 1, d, d, 200)
        reg.put(a, down, up)
    asg = np.repeat(np.arange(4, dtype=np.int32), 24)
    plan = atmm.BypassPlan(reg, asg)
    ref = atmm.BypassPlan(reg, asg)
    ref.set_overlap(False)
    x = torch.empty(asg.size, d, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y = torch.empty(asg.size, d, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y2 = y.clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            plan.apply(x, y, stream=s)
            ref.apply(x, y2, stream=s)
    s.synchronize()
    assert torch.equal(y, y2)
