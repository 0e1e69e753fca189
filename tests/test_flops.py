"""Algorithmic FLOP accounting (flops.hpp:10-24), restating the reference's
KATs: test_atmm.cpp:118-125 (2mnk), test_batch.cpp:96-128 (bypass = sum over
segments of ns * 2 * d * r * 2, padding-free, heterogeneous ranks at their own
rank), test_model.cpp:179-219 (merged forward = base cost; mixture guests pay
own + cancel).  The host-only checks run on CPU; the counter around device
calls needs a GPU."""
import numpy as np
import pytest


def test_bypass_flops_equal_ranks_padding_free(atmm):
    d, r = 64, 8
    counts = []
    for num_adapters in (1, 4):
        assignment = [i % num_adapters for i in range(8)]
        f = atmm.bypass_flops(assignment, {a: r for a in range(num_adapters)}, d)
        assert f == 8 * 2 * d * r * 2
        counts.append(f)
    assert counts[0] == counts[1]


def test_bypass_flops_heterogeneous_ranks(atmm):
    d = 64
    f = atmm.bypass_flops([1, 2, 1, 2, 1, 2], {1: 4, 2: 32}, d)
    assert f == 3 * 2 * d * 4 * 2 + 3 * 2 * d * 32 * 2


def test_bypass_flops_rectangular_and_unknown(atmm):
    assert atmm.bypass_flops([5, 5, 5], {5: 16}, 512, 384) == 3 * 2 * 16 * (512 + 384)
    with pytest.raises(atmm.UnknownAdapterError):
        atmm.bypass_flops([1, 2], {1: 8}, 64)
    with pytest.raises(atmm.ConfigError):
        atmm.bypass_flops([], {1: 8}, 64)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_bench_flops_match_the_accounting(atmm, name):
    """bench.py's FLOPs (workloads.flops) are the reference's accounting."""
    from paper_2411_00915_b200.workloads import bypass_config

    w = bypass_config(name)
    assert w.flops() == atmm.bypass_flops(w.assignment, w.ranks, w.d_in, w.d_out)
    if name == "cfg2":
        assert w.flops() == 134_217_728  # 512 * 2 * 4096 * 16 * 2


def test_merge_flops_formula():
    from paper_2411_00915_b200.workloads import MergeWorkload

    mw = MergeWorkload()
    assert mw.flops() == 32 * (2 * 4096 * 11008 * 64 + 4096 * 11008)


@pytest.mark.gpu
def test_device_counter_gemm_bypass_merge(gpu, atmm, oracle):
    import torch

    a = np.random.default_rng(5).uniform(-1, 1, (10, 20)).astype(np.float32)
    b = np.random.default_rng(6).uniform(-1, 1, (20, 30)).astype(np.float32)
    sc = atmm.FlopScope()
    atmm.atmm_multiply(a, b, (16, 16, 16, 16, 16, 16))
    assert sc.elapsed() == 2 * 10 * 20 * 30  # test_atmm.cpp:118-125

    d = 64
    reg = atmm.AdapterRegistry(1, d, d)
    rng = np.random.default_rng(1)
    for a_id, r in {1: 4, 2: 32}.items():
        reg.put(a_id, rng.uniform(-0.3, 0.3, (d, r)).astype(np.float32), rng.uniform(-0.3, 0.3, (r, d)).astype(np.float32))
    assignment = [1, 2, 1, 2, 1, 2]
    x = rng.uniform(-1, 1, (6, d)).astype(np.float32)
    sc = atmm.FlopScope()
    atmm.run_bypass(reg, x, assignment)
    assert sc.elapsed() == 3 * 2 * d * 4 * 2 + 3 * 2 * d * 32 * 2  # test_batch.cpp:120-127

    plan = atmm.BypassPlan(reg, assignment)
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    yt = torch.zeros(6, d, device="cuda", dtype=torch.float32)
    sc = atmm.FlopScope()
    plan.apply(xt, yt)
    plan.apply(xt, yt)
    assert sc.elapsed() == 2 * (3 * 2 * d * 4 * 2 + 3 * 2 * d * 32 * 2)

    W = torch.zeros(1, d, d, device="cuda", dtype=torch.float32)
    sc = atmm.FlopScope()
    atmm.merge_layers_into(reg, 2, W)
    assert sc.elapsed() == 2 * d * d * 32  # delta_w_into, model.hpp:124
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_device_counter_forward_modes(gpu, atmm):
    """test_model.cpp:179-219: merged forward = base cost exactly; mixture
    guests pay their own bypass plus the cancel branch, hosts pay nothing."""
    import torch

    L, d, r, n = 2, 64, 8, 4
    rng = np.random.default_rng(3)
    reg = atmm.AdapterRegistry(L, d, d)
    for a_id in (1, 2):
        reg.put(a_id, rng.uniform(-0.3, 0.3, (L, d, r)).astype(np.float32),
                rng.uniform(-0.3, 0.3, (L, r, d)).astype(np.float32))
    W = (torch.rand(L, d, d, device="cuda") * 0.2 - 0.1).to(torch.bfloat16)
    x = (torch.rand(n, d, device="cuda") * 2 - 1).to(torch.bfloat16)
    base = n * L * 2 * d * d
    sc = atmm.FlopScope()
    atmm.forward_merged(W, x)
    assert sc.elapsed() == base
    sc = atmm.FlopScope()
    atmm.forward_mixture(W, x, [1, 1, 1, 1], reg, merged_id=1)
    assert sc.elapsed() == base
    sc = atmm.FlopScope()
    atmm.forward_mixture(W, x, [1, 2, 1, 2], reg, merged_id=1)
    bypass_once = 2 * L * 2 * d * r * 2
    assert sc.elapsed() == base + 2 * bypass_once
    sc = atmm.FlopScope()
    atmm.forward_unmerged(W, x, [1, 2, 1, 2], reg)
    assert sc.elapsed() == base + n * L * 2 * d * r * 2
    torch.cuda.synchronize()
