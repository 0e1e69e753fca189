"""GPU parity of merge / unmerge / delta_w / atmm_multiply against the oracle.

Mirrors test_model.cpp (delta_w KATs, merge in place, toy 2x2 merge, round
trip) and test_atmm.cpp / acceptance.cpp criterion 1 (ATMM vs oracle on
random shapes).  Tolerance: 1e-2 * max(1, max|ref|) (bf16 operands).
"""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


def test_delta_w_rank1_kat(gpu, atmm):
    """test_model.cpp:27-46: unit rank-1 factors -> single 1.0 at (3, 5)."""
    d = 64
    down = np.zeros((d, 1), np.float32)
    down[3, 0] = 1.0
    up = np.zeros((1, d), np.float32)
    up[0, 5] = 1.0
    reg = atmm.AdapterRegistry(1, d, d)
    reg.put(9, down, up)
    dw = atmm.delta_w(reg, 9, 0)
    assert dw[3, 5] == 1.0
    assert np.max(np.abs(dw)) == 1.0
    assert np.sum(np.abs(dw)) == 1.0


def test_delta_w_zero_and_random(gpu, atmm, oracle):
    reg = atmm.AdapterRegistry(1, 64, 64)
    reg.put(8, np.zeros((64, 4), np.float32), np.zeros((4, 64), np.float32))
    assert np.max(np.abs(atmm.delta_w(reg, 8, 0))) == 0.0
    down, up = oracle.adapter_random(123, 1, 32, 4)
    down, up = oracle.round_bf16(down), oracle.round_bf16(up)
    reg2 = atmm.AdapterRegistry(1, 32, 32)
    reg2.put(7, down, up)
    got = atmm.delta_w(reg2, 7, 0)
    want = oracle.gemm_reference_f64(down[0], up[0])
    assert np.max(np.abs(got - want)) <= 1e-4 * max(1.0, np.max(np.abs(want)))  # exact bf16 products, fp32 sum
    with pytest.raises(atmm.ConfigError):
        atmm.delta_w(reg2, 7, 5)


def test_toy_2x2_merge(gpu, atmm):
    """test_model.cpp:102-119: identity W, delta single 1 at (0,0) -> W'(0,0) = 2."""
    import torch

    d = 16
    w = torch.eye(d, dtype=torch.float32, device="cuda")
    down = np.zeros((d, 1), np.float32)
    up = np.zeros((1, d), np.float32)
    down[0, 0] = 1.0
    up[0, 0] = 1.0
    reg = atmm.AdapterRegistry(1, d, d)
    reg.put(1, down, up)
    atmm.merge_into(reg, 1, 0, w, sign=+1.0)
    torch.cuda.synchronize()
    w = w.cpu().numpy()
    assert w[0, 0] == 2.0 and w[1, 1] == 1.0 and w[0, 1] == 0.0


@pytest.mark.parametrize("d_in,d_out,r", [(64, 64, 8), (256, 384, 16), (1000, 777, 48), (4096, 11008, 64)])
def test_merge_fp32_matches_oracle(gpu, atmm, oracle, d_in, d_out, r):
    import torch

    rng = oracle.rng(d_in + r)
    s = 1.0 / np.sqrt(np.float32(r))
    down = oracle.round_bf16(oracle.random_matrix(rng, d_in, r, -s, s))
    up = oracle.round_bf16(oracle.random_matrix(rng, r, d_out, -s, s))
    w0 = oracle.random_matrix(rng, d_in, d_out, -0.05, 0.05)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    reg.put(1, down, up)
    wt = torch.from_numpy(w0).cuda()
    atmm.merge_into(reg, 1, 0, wt, sign=+1.0)
    torch.cuda.synchronize()
    got = wt.cpu().numpy()
    rows = np.arange(d_in) if d_in <= 1024 else np.random.default_rng(0).choice(d_in, 96, replace=False)
    dw = oracle.gemm_reference_f64(down[rows], up)
    want = w0[rows].astype(np.float64) + dw
    assert np.max(np.abs(got[rows] - want)) <= 1e-4 * max(1.0, np.max(np.abs(want)))
    # unmerge restores W (round trip on fp32 weights)
    atmm.merge_into(reg, 1, 0, wt, sign=-1.0)
    torch.cuda.synchronize()
    back = wt.cpu().numpy()
    assert np.max(np.abs(back - w0)) <= 1e-6 * 10


def test_merge_bf16_weights(gpu, atmm, oracle):
    import torch

    d_in, d_out, r = 512, 640, 64
    rng = oracle.rng(3)
    s = 1.0 / np.sqrt(np.float32(r))
    down = oracle.round_bf16(oracle.random_matrix(rng, d_in, r, -s, s))
    up = oracle.round_bf16(oracle.random_matrix(rng, r, d_out, -s, s))
    w0 = oracle.round_bf16(oracle.random_matrix(rng, d_in, d_out, -0.05, 0.05))
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    reg.put(1, down, up, scale=0.5)
    wt = torch.from_numpy(w0).to("cuda", torch.bfloat16)
    atmm.merge_into(reg, 1, 0, wt, sign=-1.0)
    torch.cuda.synchronize()
    got = wt.float().cpu().numpy()
    want = w0.astype(np.float64) - 0.5 * oracle.gemm_reference_f64(down, up)
    assert np.max(np.abs(got - want)) <= tol_for(want)


def test_round_trip_100_cycles_fp32(gpu, atmm, oracle):
    """acceptance.cpp:177-211: 100 merge/unmerge cycles, drift <= 1e-4 max(1, max|W|),
    address-stable (in place on the same tensor)."""
    import torch

    L, d, r = 4, 256, 64
    w = oracle.model_random(44, L, d)
    down, up = oracle.adapter_random(45, L, d, r)
    reg = atmm.AdapterRegistry(L, d, d)
    reg.put(1, down, up)
    wt = torch.from_numpy(w).cuda()
    ptrs = [wt[l].data_ptr() for l in range(L)]
    for _ in range(100):
        for l in range(L):
            atmm.merge_into(reg, 1, l, wt[l], sign=+1.0)
        for l in range(L):
            atmm.merge_into(reg, 1, l, wt[l], sign=-1.0)
    torch.cuda.synchronize()
    assert [wt[l].data_ptr() for l in range(L)] == ptrs
    drift = float(np.max(np.abs(wt.cpu().numpy() - w)))
    assert drift <= 1e-4 * max(1.0, float(np.max(np.abs(w))))


@pytest.mark.parametrize("seed", range(6))
def test_atmm_multiply_random_shapes(gpu, atmm, oracle, seed):
    """test_atmm.cpp:21-35 / acceptance criterion 1, bf16 tolerance."""
    rng = np.random.default_rng(seed)
    m, k, n = (int(v) for v in rng.integers(1, 300, 3))
    a = oracle.round_bf16(rng.uniform(-1, 1, (m, k)).astype(np.float32))
    b = oracle.round_bf16(rng.uniform(-1, 1, (k, n)).astype(np.float32))
    got = atmm.atmm_multiply(a, b, (64, 32, 32, 32, 32, 32))
    want = oracle.gemm_reference_f64(a, b)
    assert np.max(np.abs(got - want)) <= tol_for(want)


def test_atmm_multiply_kat_and_errors(gpu, atmm):
    got = atmm.atmm_multiply([[1, 2], [3, 4]], [[5, 6], [7, 8]], (16, 16, 16, 16, 16, 16))
    assert np.array_equal(got, np.asarray([[19, 22], [43, 50]], np.float32))
    with pytest.raises(atmm.ShapeError):
        atmm.atmm_multiply(np.zeros((4, 5)), np.zeros((4, 5)), (16, 16, 16, 16, 16, 16))
    with pytest.raises(atmm.ConfigError):
        atmm.atmm_multiply(np.zeros((4, 5)), np.zeros((5, 4)), (24, 16, 16, 8, 16, 16))


@pytest.mark.parametrize("w_dtype", ["f32", "bf16"])
@pytest.mark.parametrize("d_in,d_out,pad", [(200, 136, 8), (300, 520, 0), (128, 4104, 24)])
def test_merge_tma_staged_strided(gpu, atmm, oracle, w_dtype, d_in, d_out, pad):
    """TMA-staged W path: partial 128-row tiles, partial slabs, a row stride
    wider than d_out; the padding columns must stay untouched."""
    import torch

    r = 32
    rng = oracle.rng(d_in * 7 + d_out)
    s = 1.0 / np.sqrt(np.float32(r))
    down = oracle.round_bf16(oracle.random_matrix(rng, d_in, r, -s, s))
    up = oracle.round_bf16(oracle.random_matrix(rng, r, d_out, -s, s))
    base = oracle.random_matrix(rng, d_in, d_out + pad, -0.05, 0.05)
    if w_dtype == "bf16":
        base = oracle.round_bf16(base)
    reg = atmm.AdapterRegistry(1, d_in, d_out)
    reg.put(1, down, up, scale=2.0)
    dt = torch.float32 if w_dtype == "f32" else torch.bfloat16
    full = torch.from_numpy(base).to("cuda", dt)
    view = full[:, :d_out]
    atmm.merge_into(reg, 1, 0, view, sign=+1.0)
    torch.cuda.synchronize()
    got = full.float().cpu().numpy()
    want = base[:, :d_out].astype(np.float64) + 2.0 * oracle.gemm_reference_f64(down, up)
    tol = 1e-4 * max(1.0, np.max(np.abs(want))) if w_dtype == "f32" else tol_for(want)
    assert np.max(np.abs(got[:, :d_out] - want)) <= tol
    assert np.array_equal(got[:, d_out:], base[:, d_out:].astype(np.float32))


@pytest.mark.parametrize("w_dtype", ["f32", "bf16"])
def test_merge_all_layers_one_launch(gpu, atmm, oracle, w_dtype):
    """The mode switch's one-shot merge of every layer (model.hpp:144-188) in
    one launch equals the per-layer merges; unmerge restores W (fp32)."""
    import torch

    L, d_in, d_out, r = 5, 384, 520, 48
    rng = oracle.rng(77)
    s = 1.0 / np.sqrt(np.float32(r))
    down = oracle.round_bf16(oracle.random_matrix(rng, L * d_in, r, -s, s).reshape(L, d_in, r))
    up = oracle.round_bf16(oracle.random_matrix(rng, L * r, d_out, -s, s).reshape(L, r, d_out))
    w0 = oracle.random_matrix(rng, L * d_in, d_out, -0.05, 0.05).reshape(L, d_in, d_out)
    if w_dtype == "bf16":
        w0 = oracle.round_bf16(w0)
    reg = atmm.AdapterRegistry(L, d_in, d_out)
    reg.put(1, down, up)
    dt = torch.float32 if w_dtype == "f32" else torch.bfloat16
    wa = torch.from_numpy(w0).to("cuda", dt)
    wb = wa.clone()
    atmm.merge_layers_into(reg, 1, wa, sign=+1.0)
    for l in range(L):
        atmm.merge_into(reg, 1, l, wb[l], sign=+1.0)
    torch.cuda.synchronize()
    assert torch.equal(wa, wb)
    got = wa.float().cpu().numpy()
    for l in range(L):
        want = w0[l].astype(np.float64) + oracle.gemm_reference_f64(down[l], up[l])
        tol = 1e-4 * max(1.0, np.max(np.abs(want))) if w_dtype == "f32" else tol_for(want)
        assert np.max(np.abs(got[l] - want)) <= tol
    # a sub-range of layers on a strided view, then unmerge everything
    if w_dtype == "f32":
        atmm.merge_layers_into(reg, 1, wa[1:4], sign=-1.0, layer0=1)
        atmm.merge_layers_into(reg, 1, wa[0:1], sign=-1.0, layer0=0)
        atmm.merge_layers_into(reg, 1, wa[4:5], sign=-1.0, layer0=4)
        torch.cuda.synchronize()
        assert np.max(np.abs(wa.cpu().numpy() - w0)) <= 1e-5
    with pytest.raises(atmm.ConfigError):
        atmm.merge_layers_into(reg, 1, wa[0:2], layer0=4)
