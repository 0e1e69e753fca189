#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the reference itself.

Runs the UNMODIFIED reference (oracle/_ref/libloraserve_ref.so, built by
`make -C oracle` from /root/reference/proj/include) on small seeded cases and
stores inputs + outputs as .npz, so the oracle (and the product) can be pinned
against reference outputs even where the reference is not mounted.

    python tests/golden/make_golden.py
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402


def main():
    ref = Reference()
    out = {}

    # RNG stream (random.hpp:14-20 via std::uniform_real_distribution<float>)
    out["rng_seed7_u11"] = ref.fill_uniform(7, 4096, -1.0, 1.0)
    out["rng_seed123_s"] = ref.fill_uniform(123, 1024, -0.25, 0.25)

    # LoraAdapter::random (adapter.hpp:53-73)
    down, up = ref.adapter_random(3, 2, 48, 8, 903)
    out["adapter_id3_L2_d48_r8_seed903_down"] = down
    out["adapter_id3_L2_d48_r8_seed903_up"] = up

    # plan_batch routing (batch.hpp:28-42), incl. the test_batch.cpp KATs
    cases = {"same": [3, 3, 3], "interleaved": [7, 2, 7, 2], "distinct": [5, 1, 9],
             "random64": list(np.random.default_rng(5).integers(0, 9, 64).astype(int))}
    for name, a in cases.items():
        seg, off, rows = ref.plan_batch(a)
        out[f"plan_{name}_assignment"] = np.asarray(a, np.int32)
        out[f"plan_{name}_seg"] = seg
        out[f"plan_{name}_off"] = off
        out[f"plan_{name}_rows"] = rows

    # run_bypass (batch.hpp:48-81) on a mixed batch, d = 48, ranks {8, 16, 4}
    d, n = 48, 11
    adapters = {}
    for a, r in {1: 8, 2: 16, 5: 4}.items():
        dn, u = ref.adapter_random(a, 1, d, r, 900 + a)
        adapters[a] = (dn[0], u[0])
        out[f"bypass_down_{a}"] = dn[0]
        out[f"bypass_up_{a}"] = u[0]
    x = ref.fill_uniform(77, n * d).reshape(n, d)
    assignment = np.asarray([1, 2, 5, 1, 1, 2, 5, 5, 2, 1, 2], np.int32)
    ctx = ref.ctx(d, adapters)
    out["bypass_x"] = x
    out["bypass_assignment"] = assignment
    out["bypass_out"] = ctx.run_bypass(x, assignment)

    # atmm_multiply_into (atmm.hpp:111-142) on awkward shapes and configs
    rng = np.random.default_rng(11)
    for i, (m, k, nn, cfg) in enumerate([(33, 47, 21, (32, 16, 32, 16, 16, 16)),
                                         (65, 17, 40, (64, 32, 32, 32, 32, 32)),
                                         (130, 70, 60, (32, 32, 32, 32, 32, 32))]):
        a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        b = rng.uniform(-1, 1, (k, nn)).astype(np.float32)
        out[f"gemm{i}_a"] = a
        out[f"gemm{i}_b"] = b
        out[f"gemm{i}_cfg"] = np.asarray(cfg, np.int32)
        out[f"gemm{i}_c"] = ref.atmm_multiply(a, b, cfg)
        out[f"gemm{i}_cref"] = ref.gemm_reference(a, b)

    # delta_w + add_inplace / sub_inplace (model.hpp:120-188), rectangular
    rng = np.random.default_rng(12)
    down = rng.uniform(-0.25, 0.25, (40, 16)).astype(np.float32)
    up = rng.uniform(-0.25, 0.25, (16, 56)).astype(np.float32)
    w = rng.uniform(-0.05, 0.05, (40, 56)).astype(np.float32)
    out["merge_down"] = down
    out["merge_up"] = up
    out["merge_w"] = w.copy()
    wm = w.copy()
    ref.merge_rect(wm, down, up, +1)
    out["merge_w_merged"] = wm.copy()
    ref.merge_rect(wm, down, up, -1)
    out["merge_w_roundtrip"] = wm


    # stack forward (model.hpp:192-328): the mode-equivalence setting of
    # verify.hpp:63-100 -- L = 3, d = 64, rank 16, adapters 1 and 2, 6 rows
    L, d = 3, 64
    w = np.zeros((L, d, d), np.float32)
    ref.L.ref_model_random(L, d, 64, 2024, w.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    fwd_adapters = {}
    for a in (1, 2):
        dn, u = ref.adapter_random(a, L, d, 16, 2024 * 31 + a)
        fwd_adapters[a] = (dn, u)
        out[f"fwd_down_{a}"] = dn
        out[f"fwd_up_{a}"] = u
    x = ref.fill_uniform(2024 ^ 0xABCD, 6 * d).reshape(6, d)
    assignment = np.asarray([1, 2, 1, 2, 2, 1], np.int32)
    out["fwd_w"] = w
    out["fwd_x"] = x
    out["fwd_assignment"] = assignment
    out["fwd_unmerged"], _ = ref.forward(x, w, "unmerged", assignment, fwd_adapters)
    out["fwd_mixture"], wm = ref.forward(x, w, "mixture", assignment, fwd_adapters, merged_id=1)
    out["fwd_w_merged"] = wm
    out["fwd_merged"], _ = ref.forward(x, wm, "merged")

    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)

    # tiling-table lookups (tiling.hpp:181-199) incl. the test_tiling.cpp KATs
    entries = [((64, 256, 16), (64, 32, 32, 32, 32, 32)), ((128, 256, 16), (128, 64, 64, 32, 32, 32)),
               ((256, 4096, 32), (64, 32, 32, 32, 32, 32)), ((8192, 4096, 128), (64, 64, 64, 32, 64, 64))]
    dflt = (32, 32, 32, 32, 32, 32)
    keys = np.asarray([e[0] for e in entries], np.int32).reshape(-1)
    cfgs = np.asarray([e[1] for e in entries], np.int32).reshape(-1)
    queries = [(33, 256, 16), (90, 256, 16), (96, 256, 16), (200, 256, 16), (64, 128, 16), (256, 4096, 32),
               (8192, 4096, 128), (8000, 4096, 128), (1, 256, 16), (160, 256, 16)]
    res = []
    for (m, k, nn) in queries:
        o = np.zeros(6, np.int32)
        ref.L.ref_table_lookup(keys.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                               cfgs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(entries),
                               np.asarray(dflt, np.int32).ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), m, k, nn,
                               o.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        res.append({"m": m, "k": k, "n": nn, "config": [int(v) for v in o]})
    buckets = {str(m): int(ref.L.ref_m_bucket_of(m)) for m in (0, 1, 31, 32, 33, 64, 65, 4095, 4096, 4097)}
    counts = {f"{b}_{w}": int(ref.L.ref_candidate_count(b, w)) for b, w in [(1 << 20, 4), (3 * 16 * 16 * 4, 4),
                                                                             (1 << 20, 8), (1 << 16, 4)]}
    with open(os.path.join(HERE, "tiling_vectors.json"), "w") as f:
        json.dump({"entries": [{"key": list(e[0]), "config": list(e[1])} for e in entries], "default": list(dflt),
                   "lookups": res, "m_bucket_of": buckets, "candidate_counts": counts}, f, indent=1)
    print("wrote", os.path.join(HERE, "reference_vectors.npz"), "and tiling_vectors.json")


if __name__ == "__main__":
    main()
