"""Mode-state contract on device (model.hpp:144-188, serving.hpp:38-74),
restating test_model.cpp:62-100 ("merge applies deltas in place and flips
mode": double merge -> ModeError, unmerge of the other adapter -> ModeError)
and the minimal mode_switch sequence (merged -> mixture of the same adapter
touches no weights)."""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


def _setup(atmm, oracle, L=3, d=256, ranks=(16, 8), dtype="float32"):
    import torch

    reg = atmm.AdapterRegistry(L, d, d)
    facs = {}
    for i, r in enumerate(ranks, start=1):
        down, up = oracle.adapter_random(2000 + i, L, d, r)
        down, up = oracle.round_bf16(down), oracle.round_bf16(up)
        reg.put(i, down, up)
        facs[i] = (down, up)
    w0 = oracle.model_random(77, L, d)
    W = torch.from_numpy(w0).to("cuda", getattr(torch, dtype)).contiguous()
    return reg, facs, w0, W


def test_merge_flips_mode_and_rejects_misuse(gpu, atmm, oracle):
    import torch

    reg, facs, w0, W = _setup(atmm, oracle)
    addr = W.data_ptr()
    st = atmm.ModelState(reg, W)
    assert st.mode == "unmerged" and st.merged_adapter == -1
    st.merge(1)
    torch.cuda.synchronize()
    assert st.mode == "merged" and st.merged_adapter == 1
    assert W.data_ptr() == addr  # in place, no reallocation
    got = W.cpu().numpy()
    for l in range(w0.shape[0]):
        want = w0[l].astype(np.float64) + facs[1][0][l].astype(np.float64) @ facs[1][1][l].astype(np.float64)
        assert np.max(np.abs(got[l] - want)) <= tol_for(want)
    with pytest.raises(atmm.ModeError):
        st.merge(1)  # double merge is rejected by contract
    with pytest.raises(atmm.ModeError):
        st.merge(2)
    with pytest.raises(atmm.ModeError):
        st.unmerge(2)  # unmerging a different adapter is an identity error
    assert st.weight_writes == 1  # rejected calls wrote nothing
    st.unmerge(1)
    torch.cuda.synchronize()
    assert st.mode == "unmerged"
    back = W.cpu().numpy()
    # the same dW is added then subtracted in fp32: two roundings at |W + dW|
    bound = 2 * 2.0 ** -24 * float(np.max(np.abs(got))) + 1e-7
    assert float(np.max(np.abs(back - w0))) <= bound
    with pytest.raises(atmm.ModeError):
        st.unmerge(1)


def test_mode_switch_minimal_sequence(gpu, atmm, oracle):
    import torch

    reg, facs, w0, W = _setup(atmm, oracle, dtype="float32")
    st = atmm.ModelState(reg, W)
    assert st.mode_switch("merged", 1) == 1
    assert (st.mode, st.merged_adapter) == ("merged", 1)
    snap = W.clone()
    assert st.mode_switch("mixture", 1) == 0  # merged -> mixture: no weight writes
    torch.cuda.synchronize()
    assert st.mode == "mixture" and torch.equal(W, snap)
    assert st.mode_switch("merged", 1) == 0
    assert st.mode_switch("mixture", 2) == 2  # unmerge 1, merge 2
    assert (st.mode, st.merged_adapter) == ("mixture", 2)
    torch.cuda.synchronize()
    got = W.cpu().numpy()
    for l in range(w0.shape[0]):
        want = w0[l].astype(np.float64) + facs[2][0][l].astype(np.float64) @ facs[2][1][l].astype(np.float64)
        assert np.max(np.abs(got[l] - want)) <= tol_for(want)
    assert st.mode_switch("unmerged") == 1
    assert st.mode_switch("unmerged") == 0
    with pytest.raises(atmm.ModeError):
        st.mode_switch("merged")  # needs a target adapter
    with pytest.raises(atmm.UnknownAdapterError):
        st.mode_switch("merged", 99)
    with pytest.raises(atmm.ModeError):
        st.set_mixture(1)  # nothing merged
    st.merge(1)
    with pytest.raises(atmm.ModeError):
        st.set_mixture(2)  # the delora branch must be the merged adapter
    st.set_mixture(1)
    assert st.mode == "mixture"
    torch.cuda.synchronize()


def test_mode_switch_bf16_weights_all_layers_one_launch(gpu, atmm, oracle):
    import torch

    reg, facs, w0, W = _setup(atmm, oracle, L=4, d=512, ranks=(64, 16), dtype="bfloat16")
    st = atmm.ModelState(reg, W)
    sc = atmm.FlopScope()
    assert st.mode_switch("merged", 2) == 1
    assert sc.elapsed() == 4 * 2 * 512 * 512 * 16
    torch.cuda.synchronize()
    got = W.float().cpu().numpy()
    wb = oracle.round_bf16(w0)
    for l in range(4):
        want = wb[l].astype(np.float64) + facs[2][0][l].astype(np.float64) @ facs[2][1][l].astype(np.float64)
        assert np.max(np.abs(got[l] - want)) <= tol_for(want)
