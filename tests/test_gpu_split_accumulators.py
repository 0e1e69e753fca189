"""Split path (atmm_shrink_kernel + atmm_expand_kernel) with full 128-row
tiles, where the expand's two TMEM accumulators are G x 128 columns each, and
rank-chunk passes that reuse a plan's scratch on one stream.

Regression for two ordering bugs that only showed under particular timings:
the expand's second accumulator overlapping the first when G x rows16 > 128
(odd output columns of one item overwritten by the next item's MMA), and the
per-tile mid readiness counters.  Every apply here gets NEW inputs (the
previous apply's mid would otherwise hide a read-before-ready) and is checked
against the oracle; reruns on the same inputs must be bit-identical.
"""
import numpy as np
import pytest

from conftest import path_table, tol_for

pytestmark = pytest.mark.gpu


def _registry(atmm, oracle, d, ranks, seed):
    reg = atmm.AdapterRegistry(1, d, d)
    facs = {}
    rng = oracle.rng(seed)
    for a, r in ranks.items():
        s = 1.0 / np.sqrt(np.float32(r))
        down = oracle.round_bf16(oracle.random_matrix(rng, d, r, -s, s))
        up = oracle.round_bf16(oracle.random_matrix(rng, r, d, -s, s))
        reg.put(a, down[None], up[None])
        facs[a] = (down, up)
    return reg, facs


@pytest.mark.parametrize("ranks,rows", [
    ({0: 16, 1: 32, 2: 64, 3: 64}, 128),     # G = 2, 128-row tiles: 2 x 256 accumulator columns
    ({0: 48, 1: 16}, 112),                    # G = 2, rows16 = 112
    ({0: 300, 1: 64}, 200),                   # rank chunks: passes of r_pad 128 (G = 1) and 48 (G = 2)
])
@pytest.mark.parametrize("ydt", ["bf16", "f32"])
@pytest.mark.parametrize("order", ["shuffled", "sorted", "runs"])
def test_split_fresh_inputs_every_apply(gpu, atmm, oracle, ranks, rows, ydt, order):
    """order: shuffled rows (every tile gathered row by row), sorted (every
    tile's rows consecutive: X / Y by TMA boxes, TileDesc::x_row0), runs
    (requests of 40 consecutive rows interleaved: some tiles of each kind)."""
    import torch

    d = 1024
    reg, facs = _registry(atmm, oracle, d, ranks, 11)
    asg = np.repeat(np.asarray(sorted(ranks), np.int32), rows)
    if order == "shuffled":
        asg = asg[np.random.default_rng(3).permutation(asg.size)]
    elif order == "runs":
        runs = [asg[i:i + 40] for i in range(0, asg.size, 40)]
        perm = np.random.default_rng(3).permutation(len(runs))
        asg = np.concatenate([runs[i] for i in perm])
    n = asg.size
    plan = atmm.BypassPlan(reg, asg, path_table(atmm, asg, ranks, d, d, "split"))
    assert {g["path_bf16"] for g in plan.describe()} == {"split"}
    dt = torch.bfloat16 if ydt == "bf16" else torch.float32
    rng = oracle.rng(7)
    for step in range(6):
        x = oracle.round_bf16(oracle.random_matrix(rng, n, d))
        y0 = oracle.round_bf16(oracle.random_matrix(rng, n, d))
        xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
        outs = []
        for _ in range(2):
            yt = torch.from_numpy(y0).to("cuda", dt)
            plan.apply(xt, yt, layer=0)
            outs.append(yt)
        torch.cuda.synchronize()
        want = y0.astype(np.float64) + oracle.bypass_rows_f64(x, asg, facs)
        got = outs[0].float().cpu().numpy()
        err = float(np.max(np.abs(got - want)))
        assert err <= tol_for(want), (step, err)
        assert torch.equal(outs[0], outs[1]), f"step {step}: reruns differ"


@pytest.mark.parametrize("rows,rank", [(16, 16), (64, 16), (100, 48), (128, 16), (128, 64), (128, 128)])
def test_expand_tmem_holds_two_accumulators(gpu, atmm, oracle, rows, rank):
    """Structural: the expand's TMEM allocation holds both accumulators
    (2 x G x rows16 columns), and shared memory is padded so the expand CTAs
    that can share an SM fit in its 512 columns (a CTA blocked in
    tcgen05.alloc would hold back the reduction share other CTAs wait for)."""
    d = 1024
    reg, _ = _registry(atmm, oracle, d, {0: rank, 1: rank}, 5)
    asg = np.repeat(np.asarray([0, 1], np.int32), rows)
    plan = atmm.BypassPlan(reg, asg, path_table(atmm, asg, {0: rank, 1: rank}, d, d, "split"))
    smem_per_sm = 233472
    for g in plan.describe():
        sp = g["split"]
        assert sp is not None
        for di, gg in ((0, sp["g_bf16"]), (1, 1)):
            cols = sp["etmem"][di]
            assert cols >= 2 * gg * sp["rows16"] and cols <= 512, (sp, di)
            co = smem_per_sm // (sp["smem_e"][di] + 1024)
            assert co * cols <= 512, (sp, di, co)


@pytest.mark.parametrize("swap", ["put", "put_async"])
def test_split_up_copy_follows_adapter_replacement(gpu, atmm, oracle, swap):
    """256-column expand items read an MMA-ordered copy of up^T made when a
    split plan first uses the slot (Slot::up_t2): replacing the adapter (put,
    or put_async on a stream) must never leave a plan reading the old copy."""
    import torch

    d = 1024
    ranks = {0: 32, 1: 64}
    reg, facs = _registry(atmm, oracle, d, ranks, 21)
    asg = np.repeat(np.asarray([0, 1], np.int32), 128)
    asg = asg[np.random.default_rng(2).permutation(asg.size)]
    n = asg.size
    tbl = path_table(atmm, asg, ranks, d, d, "split")
    rng = oracle.rng(5)
    x = oracle.round_bf16(oracle.random_matrix(rng, n, d))
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)

    def check(plan, facs):
        y0 = oracle.round_bf16(oracle.random_matrix(rng, n, d))
        yt = torch.from_numpy(y0).to("cuda", torch.bfloat16)
        plan.apply(xt, yt, layer=0)
        torch.cuda.synchronize()
        want = y0.astype(np.float64) + oracle.bypass_rows_f64(x, asg, facs)
        assert float(np.max(np.abs(yt.float().cpu().numpy() - want))) <= tol_for(want)

    plan = atmm.BypassPlan(reg, asg, tbl)
    check(plan, facs)
    # replace adapter 1 (same rank) with new factors
    r = ranks[1]
    s = 1.0 / np.sqrt(np.float32(r))
    down = oracle.round_bf16(oracle.random_matrix(rng, d, r, -s, s))
    up = oracle.round_bf16(oracle.random_matrix(rng, r, d, -s, s))
    if swap == "put":
        reg.put(1, down[None], up[None])
    else:
        st = torch.cuda.Stream()
        reg.put_async(1, down[None], up[None], stream=st)
        st.synchronize()
    facs = dict(facs)
    facs[1] = (down, up)
    plan2 = atmm.BypassPlan(reg, asg, tbl)
    check(plan2, facs)
