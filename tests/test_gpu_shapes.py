"""Any hidden size through the device API (the reference takes any
d_in / d_out, adapter.hpp / batch.hpp): X rows that are not 16-byte aligned
(d_in % 8 != 0, or an offset view) are staged into a padded copy, Y rows that
are not vector aligned take the general fused kernel.  Oracle parity with
the north-star tolerance, bit-exact reruns."""
import numpy as np
import pytest

from conftest import tol_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ydt", ["bf16", "f32"])
@pytest.mark.parametrize("d_in,d_out,ranks,lens", [
    (1003, 517, {1: 16, 2: 40}, [37, 90]),
    (77, 130, {3: 8}, [13]),
    (4099, 4095, {4: 64, 5: 16}, [40, 9]),
])
def test_odd_hidden_sizes_device_api(gpu, atmm, oracle, ydt, d_in, d_out, ranks, lens):
    import torch

    reg = atmm.AdapterRegistry(1, d_in, d_out)
    facs = {}
    rng = oracle.rng(21)
    for a, r in ranks.items():
        s = 1.0 / np.sqrt(np.float32(r))
        down = oracle.round_bf16(oracle.random_matrix(rng, d_in, r, -s, s))
        up = oracle.round_bf16(oracle.random_matrix(rng, r, d_out, -s, s))
        reg.put(a, down[None], up[None])
        facs[a] = (down, up)
    ids = sorted(ranks)
    asg = np.concatenate([np.full(n, ids[i], np.int32) for i, n in enumerate(lens)])
    asg = asg[np.random.default_rng(2).permutation(asg.size)]
    n = asg.size
    x = oracle.round_bf16(oracle.random_matrix(oracle.rng(5), n, d_in))
    y0 = oracle.round_bf16(oracle.random_matrix(oracle.rng(6), n, d_out))
    want = y0.astype(np.float64) + oracle.bypass_rows_f64(x, asg, facs)
    plan = atmm.BypassPlan(reg, asg)
    dt = torch.bfloat16 if ydt == "bf16" else torch.float32
    # a contiguous X, and an X view one element into a wider buffer (misaligned rows)
    wide = torch.zeros(n, d_in + 3, dtype=torch.bfloat16, device="cuda")
    wide[:, 1:1 + d_in] = torch.from_numpy(x).to(torch.bfloat16)
    for xt in (torch.from_numpy(x).to("cuda", torch.bfloat16), wide[:, 1:1 + d_in]):
        outs = []
        for _ in range(2):
            yt = torch.from_numpy(y0).to("cuda", dt)
            plan.apply(xt, yt)
            outs.append(yt)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1])
        got = outs[0].float().cpu().numpy()
        assert np.max(np.abs(got - want)) <= tol_for(want)
