"""GPU: a reference fixture loads into the device registry, and the async
adapter swap packs factors on device bit-identically to the host path."""
import numpy as np
import pytest

from conftest import tol_for
from test_fixture import write_reference_fixture

pytestmark = pytest.mark.gpu


def test_load_reference_fixture_matches_put(gpu, atmm, oracle, reference, tmp_path):
    import torch

    L, d, n = 2, 256, 64
    rng = np.random.default_rng(2)
    adapters = {}
    for aid, r in [(1, 16), (2, 40)]:
        adapters[aid] = (oracle.round_bf16(rng.uniform(-0.2, 0.2, (L, d, r)).astype(np.float32)),
                         oracle.round_bf16(rng.uniform(-0.2, 0.2, (L, r, d)).astype(np.float32)))
    write_reference_fixture(reference, tmp_path, L, d, adapters)
    reg_f = atmm.AdapterRegistry(L, d, d)
    assert reg_f.load_fixture(tmp_path) == 2
    reg_p = atmm.AdapterRegistry(L, d, d)
    for aid, (dn, up) in adapters.items():
        reg_p.put(aid, dn, up)
    assignment = np.asarray([1 + i % 2 for i in range(n)], np.int32)
    x = torch.from_numpy(oracle.round_bf16(oracle.random_matrix(oracle.rng(4), n, d))).to("cuda", torch.bfloat16)
    for layer in range(L):
        ya, yb = torch.zeros(n, d, device="cuda"), torch.zeros(n, d, device="cuda")
        atmm.BypassPlan(reg_f, assignment).apply(x, ya, layer=layer)
        atmm.BypassPlan(reg_p, assignment).apply(x, yb, layer=layer)
        torch.cuda.synchronize()
        assert torch.equal(ya, yb)
    with pytest.raises(atmm.ShapeError):
        atmm.AdapterRegistry(L, 128, 128).load_fixture(tmp_path)


def test_put_async_matches_put(gpu, atmm, oracle):
    import torch

    L, d_in, d_out, n = 3, 512, 384, 80
    rng = np.random.default_rng(6)
    down = oracle.round_bf16(rng.uniform(-0.2, 0.2, (L, d_in, 24)).astype(np.float32))
    up = oracle.round_bf16(rng.uniform(-0.2, 0.2, (L, 24, d_out)).astype(np.float32))
    reg_a = atmm.AdapterRegistry(L, d_in, d_out)
    reg_s = atmm.AdapterRegistry(L, d_in, d_out)
    stream = torch.cuda.Stream()
    reg_a.put(7, np.zeros_like(down), np.zeros_like(up))  # replaced on the stream below
    reg_a.put_async(7, torch.from_numpy(down).pin_memory(), torch.from_numpy(up).pin_memory(), scale=0.5, stream=stream)
    reg_s.put(7, down, up, scale=0.5)
    x = torch.from_numpy(oracle.round_bf16(oracle.random_matrix(oracle.rng(8), n, d_in))).to("cuda", torch.bfloat16)
    assignment = np.full(n, 7, np.int32)
    ya, yb = torch.zeros(n, d_out, device="cuda"), torch.zeros(n, d_out, device="cuda")
    with torch.cuda.stream(stream):
        atmm.BypassPlan(reg_a, assignment).apply(x, ya, layer=2, stream=stream)
    atmm.BypassPlan(reg_s, assignment).apply(x, yb, layer=2)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)
    want = 0.5 * oracle.bypass_rows_f64(x.float().cpu().numpy(), assignment, {7: (down[2], up[2])})
    assert np.max(np.abs(ya.cpu().numpy() - want)) <= tol_for(want)
