"""Request-sharded launcher on one device: every shard of
the batch run in turn equals the unsharded bypass.

Segments are independent (run_bypass, batch.hpp:57-79), so sharding by whole
segments changes nothing a row sees on the all-to-all path (a tile's K
partials are summed in the same cluster order): bit-identical.  On the split
path the fp32 partial sums of mid follow the launch's stream-K partition,
which depends on the whole launch's work, so a shard's rows agree with the
unsharded run within the north-star tolerance (each is bit-reproducible).
Every rank holds only the adapters its shard touches.
"""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


def _setup(atmm, oracle, name, seed=11):
    from paper_2411_00915_b200.workloads import bypass_config

    w = bypass_config(name)
    rng = oracle.rng(seed)
    facs = {}
    for a, r in w.ranks.items():
        s = 1.0 / np.sqrt(np.float32(r))
        facs[a] = (oracle.round_bf16(oracle.random_matrix(rng, w.d_in, r, -s, s)),
                   oracle.round_bf16(oracle.random_matrix(rng, r, w.d_out, -s, s)))
    return w, facs


def _run(atmm, oracle, name, world, exact):
    import torch

    from paper_2411_00915_b200.sharding import ShardedBypass

    w, facs = _setup(atmm, oracle, name)
    reg = atmm.AdapterRegistry(1, w.d_in, w.d_out)
    for a, (down, up) in facs.items():
        reg.put(a, down, up)
    x = torch.empty(w.tokens, w.d_in, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y0 = torch.empty(w.tokens, w.d_out, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    y_full = y0.clone()
    atmm.BypassPlan(reg, w.assignment).apply(x, y_full)
    y_glob = y0.clone()
    y_loc = y0.clone()
    covered = np.zeros(w.tokens, bool)
    for rank in range(world):
        sb = ShardedBypass(w.assignment, w.ranks, w.d_in, w.d_out, world, rank,
                           factors=lambda a: (facs[a][0][None], facs[a][1][None]))
        # only the shard's adapters are resident
        for a in w.ranks:
            assert (a in sb.registry) == (a in sb.shard.adapters)
        assert not covered[sb.rows].any()
        covered[sb.rows] = True
        sb.apply_global(x, y_glob)
        rows = torch.from_numpy(sb.rows).to("cuda")
        xl = x.index_select(0, rows)
        yl = y0.index_select(0, rows)
        sb.apply_local(xl, yl)
        y_loc.index_copy_(0, rows, yl)
    torch.cuda.synchronize()
    assert covered.all()
    assert torch.equal(y_glob, y_loc), "in-place (row-mapped) and staged shard runs must agree bit for bit"
    if exact:
        assert torch.equal(y_glob, y_full), "sharded == unsharded, bit for bit"
    pick = np.random.default_rng(world).choice(w.tokens, 48, replace=False)
    xs = x[pick].float().cpu().numpy()
    want = y0[pick].float().cpu().numpy().astype(np.float64) + oracle.bypass_rows_f64(xs, w.assignment[pick], facs)
    got = y_glob[pick].float().cpu().numpy()
    assert np.max(np.abs(got - want)) <= tol_for(want)
    full = y_full.float().cpu().numpy()
    assert np.max(np.abs(y_glob.float().cpu().numpy() - full)) <= tol_for(full)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_equals_unsharded_cfg2(gpu, atmm, oracle, world):
    _run(atmm, oracle, "cfg2", world, exact=True)


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_cfg3(gpu, atmm, oracle, world):
    _run(atmm, oracle, "cfg3", world, exact=False)


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_cfg5_exact_shape(gpu, atmm, oracle, world):
    """cfg5 at its exact shape (8192 tokens x 64 adapters r64, d 5120)."""
    _run(atmm, oracle, "cfg5", world, exact=False)
