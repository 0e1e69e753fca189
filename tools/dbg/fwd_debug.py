import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2411_00915_b200 as atmm
from oracle.oracle import Oracle
o = Oracle()
def run(L, d, ranks, lens, merged_only=False, bn=None):
    import os
    if bn: os.environ["ATMM_FWD_BN"] = bn
    w = o.round_bf16(o.model_random(1, L, d))
    reg = atmm.AdapterRegistry(L, d); facs = {}
    for a, r in ranks.items():
        dn, up = o.adapter_random(a, L, d, r); dn, up = o.round_bf16(dn), o.round_bf16(up)
        reg.put(a, dn, up); facs[a] = (dn, up)
    ids = sorted(ranks)
    a = np.concatenate([np.full(n, ids[i], np.int32) for i, n in enumerate(lens)])
    a = a[np.random.default_rng(0).permutation(a.size)]
    x = o.round_bf16(o.random_matrix(o.rng(5), a.size, d))
    dev = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to("cuda", torch.bfloat16)
    if merged_only:
        want = o.forward_f64(x, w, "merged")
        got = atmm.forward_merged(dev(w), dev(x)).float().cpu().numpy()
    else:
        want = o.forward_f64(x, w, "unmerged", a, facs)
        fw = atmm.LayerForward(atmm.BypassPlan(reg, a))
        got = fw.run(dev(w), dev(x)).float().cpu().numpy()
        print("  stats", fw.stats())
    err = np.abs(got - want).max(axis=1)
    bad = np.nonzero(err > 1e-2)[0]
    print(f"L={L} d={d} ranks={ranks} lens={lens} merged={merged_only} bn={bn}: max {err.max():.4f} bad rows {bad.size}/{a.size}",
          "bad adapters", np.unique(a[bad]) if bad.size else "")
run(1, 256, {1: 16}, [10], merged_only=True)
run(1, 256, {1: 16}, [200], merged_only=True)
run(1, 256, {1: 16}, [10])
run(1, 256, {1: 16}, [200])
run(1, 256, {1: 16, 2: 32}, [60, 60])
run(1, 256, {1: 64}, [60])
run(1, 256, {1: 128}, [60])
run(1, 256, {1: 16}, [10], bn="256")
run(2, 256, {1: 16}, [10])
run(1, 1024, {1: 16}, [300])
