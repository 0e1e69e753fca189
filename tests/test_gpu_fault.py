"""The parity harness can fail: verify.hpp:62-120 check_mode_equivalence with
its constructed fault (verify.hpp:83-85, ``model.layer(0).data[0] += 0.5``
after the merge) restated on the device path.  The same check must pass on the
clean run and fail on the faulted one; likewise the bypass parity check
against the oracle fails when one adapter factor is corrupted."""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


def _mode_equivalence(atmm, oracle, inject_fault: bool, seed: int = 4):
    """verify.hpp:63-120 on device: forward_unmerged vs merged vs mixture."""
    import torch

    L, d, rank = 3, 128, 16
    reg = atmm.AdapterRegistry(L, d, d)
    for a in (1, 2):
        down, up = oracle.adapter_random(seed * 31 + a, L, d, rank)
        reg.put(a, down, up)
    W = torch.from_numpy(oracle.model_random(seed, L, d)).to("cuda", torch.bfloat16).contiguous()
    x = torch.from_numpy(oracle.random_matrix(oracle.rng(seed ^ 0xABCD), 6, d)).to("cuda", torch.bfloat16)
    assignment = [1, 2, 1, 2, 2, 1]
    st = atmm.ModelState(reg, W)
    unmerged = atmm.forward_unmerged(W, x, assignment, reg).float()
    st.merge(1)
    if inject_fault:
        W[0, 0, 0] += 0.5  # constructed fault (verify.hpp:84)
    merged = atmm.forward_merged(W, x).float()
    st.set_mixture(1)
    mixture = atmm.forward_mixture(W, x, assignment, reg, merged_id=1).float()
    torch.cuda.synchronize()
    tol = tol_for(unmerged.cpu().numpy())
    for row, a in enumerate(assignment):
        ref = merged[row] if a == 1 else unmerged[row]
        diff = float((mixture[row] - ref).abs().max())
        if diff > tol:
            return False, f"row {row} diff {diff:.3e} > tol {tol:.3e}"
        if a == 1:
            diff = float((merged[row] - unmerged[row]).abs().max())
            if diff > tol:
                return False, f"merged/unmerged mismatch at row {row} diff {diff:.3e}"
    return True, ""


def test_mode_equivalence_passes_clean_and_fails_with_injected_fault(gpu, atmm, oracle):
    ok, detail = _mode_equivalence(atmm, oracle, inject_fault=False)
    assert ok, detail
    ok, detail = _mode_equivalence(atmm, oracle, inject_fault=True)
    assert not ok, "the injected fault went undetected"
    assert "diff" in detail


def test_bypass_parity_detects_a_corrupted_factor(gpu, atmm, oracle):
    d, n = 512, 64
    down, up = oracle.adapter_random(9, 1, d, 16)
    down, up = oracle.round_bf16(down), oracle.round_bf16(up)
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(3), n, d))
    assignment = np.full(n, 7, np.int32)
    want = oracle.bypass_rows_f64(x, assignment, {7: (down[0], up[0])})
    reg = atmm.AdapterRegistry(1, d, d)
    reg.put(7, down, up)
    assert np.max(np.abs(atmm.run_bypass(reg, x, assignment) - want)) <= tol_for(want)
    bad = down.copy()
    bad[0, 5, 3] += 0.5  # one corrupted factor element
    reg.put(7, bad, up)
    assert np.max(np.abs(atmm.run_bypass(reg, x, assignment) - want)) > tol_for(want)
