"""CPU: pin the oracle (oracle/atmm_oracle.c) to the reference.

Two independent anchors:
  * tests/golden/ fixtures generated from the reference itself
    (tests/golden/make_golden.py runs oracle/_ref, the untouched reference
    headers compiled in place);
  * the reference's own known-answer tests (test_matrix.cpp, test_batch.cpp,
    test_tiling.cpp, test_model.cpp) restated here;
plus, where oracle/_ref is built, live bit-exact comparisons on random cases.
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "reference_vectors.npz"))


@pytest.fixture(scope="module")
def tiling_gold():
    with open(os.path.join(GOLD, "tiling_vectors.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------- golden ---


def test_rng_stream_matches_reference_golden(oracle, gold):
    """random.hpp:14-20 (mt19937_64 + libstdc++ uniform_real_distribution<float>)."""
    assert np.array_equal(oracle.fill_uniform(oracle.rng(7), 4096, -1.0, 1.0), gold["rng_seed7_u11"])
    assert np.array_equal(oracle.fill_uniform(oracle.rng(123), 1024, -0.25, 0.25), gold["rng_seed123_s"])


def test_adapter_random_matches_reference_golden(oracle, gold):
    """LoraAdapter::random (adapter.hpp:53-73)."""
    down, up = oracle.adapter_random(903, 2, 48, 8)
    assert np.array_equal(down, gold["adapter_id3_L2_d48_r8_seed903_down"])
    assert np.array_equal(up, gold["adapter_id3_L2_d48_r8_seed903_up"])


@pytest.mark.parametrize("name", ["same", "interleaved", "distinct", "random64"])
def test_plan_batch_matches_reference_golden(oracle, gold, name):
    seg, off, rows = oracle.plan_batch(gold[f"plan_{name}_assignment"])
    assert np.array_equal(seg, gold[f"plan_{name}_seg"])
    assert np.array_equal(off, gold[f"plan_{name}_off"])
    assert np.array_equal(rows, gold[f"plan_{name}_rows"])


def test_run_bypass_bit_exact_with_reference_golden(oracle, gold):
    """run_bypass (batch.hpp:48-81): the restated fp32 tiled ATMM reproduces
    the reference's bits exactly."""
    adapters = {a: (gold[f"bypass_down_{a}"], gold[f"bypass_up_{a}"]) for a in (1, 2, 5)}
    got = oracle.run_bypass(gold["bypass_x"], gold["bypass_assignment"], adapters)
    assert np.array_equal(got, gold["bypass_out"])


@pytest.mark.parametrize("i", range(3))
def test_atmm_multiply_bit_exact_with_reference_golden(oracle, gold, i):
    """atmm_multiply_into (atmm.hpp:111-142) and gemm_reference (matrix.hpp:109-127)."""
    a, b, cfg = gold[f"gemm{i}_a"], gold[f"gemm{i}_b"], gold[f"gemm{i}_cfg"]
    assert np.array_equal(oracle.atmm_multiply(a, b, cfg), gold[f"gemm{i}_c"])
    assert np.array_equal(oracle.gemm_reference(a, b), gold[f"gemm{i}_cref"])


def test_merge_unmerge_bit_exact_with_reference_golden(oracle, gold):
    """delta_w_into + add/sub_inplace (model.hpp:120-188)."""
    w = gold["merge_w"][None]
    down, up = gold["merge_down"][None], gold["merge_up"][None]
    merged = oracle.merge(w, down, up, +1)
    assert np.array_equal(merged[0], gold["merge_w_merged"])
    back = oracle.merge(merged, down, up, -1)
    assert np.array_equal(back[0], gold["merge_w_roundtrip"])


def test_tiling_lookup_matches_reference_golden(oracle, tiling_gold):
    entries = [(tuple(e["key"]), tuple(e["config"])) for e in tiling_gold["entries"]]
    for q in tiling_gold["lookups"]:
        got = oracle.table_lookup(entries, tiling_gold["default"], q["m"], q["k"], q["n"])
        assert list(got) == q["config"], q
    for m, b in tiling_gold["m_bucket_of"].items():
        assert oracle.m_bucket_of(int(m)) == b


# ----------------------------------------------------- reference KATs -----


def test_gemm_reference_kats(oracle):
    """test_matrix.cpp:28-43."""
    b = np.asarray([[5, 6], [7, 8]], np.float32)
    assert np.array_equal(oracle.gemm_reference(np.eye(2, dtype=np.float32), b), b)
    assert np.array_equal(oracle.gemm_reference(np.zeros((2, 2), np.float32), b), np.zeros((2, 2)))
    assert np.array_equal(oracle.gemm_reference(np.asarray([[1, 2], [3, 4]], np.float32), b),
                          np.asarray([[19, 22], [43, 50]], np.float32))


def test_plan_batch_kats(oracle):
    """test_batch.cpp:40-61."""
    seg, off, rows = oracle.plan_batch([3, 3, 3])
    assert list(seg) == [3] and list(rows) == [0, 1, 2]
    seg, off, rows = oracle.plan_batch([7, 2, 7, 2])
    assert list(seg) == [2, 7] and list(rows[off[0]:off[1]]) == [1, 3] and list(rows[off[1]:off[2]]) == [0, 2]
    seg, off, rows = oracle.plan_batch([5, 1, 9])
    assert len(seg) == 3 and all(off[i + 1] - off[i] == 1 for i in range(3))
    with pytest.raises(ValueError):
        oracle.plan_batch([])


def test_tiling_kats(oracle):
    """test_tiling.cpp:61-87 (bucketing; lookup exact / near / default / tie)."""
    assert [oracle.m_bucket_of(m) for m in (1, 32, 33, 4096)] == [32, 32, 64, 4096]
    stored, dflt = (64, 32, 32, 32, 32, 32), (32, 32, 32, 32, 32, 32)
    e = [((64, 256, 16), stored)]
    assert oracle.table_lookup(e, dflt, 33, 256, 16) == stored
    assert oracle.table_lookup(e, dflt, 90, 256, 16) == stored
    assert oracle.table_lookup(e, dflt, 200, 256, 16) == dflt
    assert oracle.table_lookup(e, dflt, 64, 128, 16) == dflt
    e.append(((128, 256, 16), (128, 64, 64, 32, 32, 32)))
    assert oracle.table_lookup(e, dflt, 96, 256, 16) == stored
    assert oracle.config_valid((64, 32, 32, 32, 32, 32))
    assert not oracle.config_valid((48, 32, 32, 16, 16, 16))
    assert not oracle.config_valid((8, 32, 32, 8, 16, 16))
    assert not oracle.config_valid((32, 32, 32, 64, 16, 16))


def test_delta_w_kats(oracle):
    """test_model.cpp:27-46: rank-1 unit factors -> single 1.0 at (3, 5)."""
    down = np.zeros((64, 1), np.float32)
    down[3, 0] = 1.0
    up = np.zeros((1, 64), np.float32)
    up[0, 5] = 1.0
    dw = oracle.delta_w(down, up)
    assert dw[3, 5] == 1.0 and np.sum(np.abs(dw)) == 1.0


def test_toy_merge_kat(oracle):
    """test_model.cpp:102-119."""
    w = np.eye(16, dtype=np.float32)[None]
    down = np.zeros((1, 16, 1), np.float32)
    up = np.zeros((1, 1, 16), np.float32)
    down[0, 0, 0] = 1.0
    up[0, 0, 0] = 1.0
    m = oracle.merge(w, down, up, +1)[0]
    assert m[0, 0] == 2.0 and m[1, 1] == 1.0 and m[0, 1] == 0.0


def test_oracle_bypass_vs_f64_rows(oracle):
    """test_batch.cpp:63-80: run_bypass vs the per-row 64-bit oracle, 1e-4 rel."""
    rng = np.random.default_rng(77)
    d = 48
    adapters = {}
    for a, r in {1: 8, 2: 16, 5: 4}.items():
        dn, u = oracle.adapter_random(900 + a, 1, d, r)
        adapters[a] = (dn[0], u[0])
    for it in range(6):
        n = 1 + it * 2
        x = rng.uniform(-1, 1, (n, d)).astype(np.float32)
        assignment = rng.choice([1, 2, 5], n).astype(np.int32)
        got = oracle.run_bypass(x, assignment, adapters)
        want = oracle.bypass_rows_f64(x, assignment, adapters)
        assert np.max(np.abs(got - want)) <= 1e-4 * max(1.0, np.max(np.abs(want)))


# ------------------------------------------- live reference comparisons ---


def test_rng_live(oracle, reference):
    for seed in (0, 1, 42, 2 ** 63 + 5):
        assert np.array_equal(oracle.fill_uniform(oracle.rng(seed), 3000), reference.fill_uniform(seed, 3000))


def test_shuffle_live(oracle, reference):
    import ctypes

    for seed, n in [(3, 10), (44, 9), (7, 1000)]:
        v = np.arange(n, dtype=np.uint64)
        h = reference.L.ref_rng_new(seed)
        ref = np.ascontiguousarray(v.copy())
        reference.L.ref_seeded_shuffle_u64(h, ref.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n)
        reference.L.ref_rng_free(h)
        assert np.array_equal(oracle.seeded_shuffle(oracle.rng(seed), v), ref)


def test_plan_batch_live(oracle, reference):
    rng = np.random.default_rng(9)
    for n in (1, 2, 17, 300, 2048):
        a = rng.integers(-5, 40, n).astype(np.int32)
        for x, y in zip(oracle.plan_batch(a), reference.plan_batch(a)):
            assert np.array_equal(x, y)


def test_atmm_multiply_live(oracle, reference):
    """acceptance.cpp criterion 1 shapes (dims 1..200) x configs: bit-exact."""
    rng = np.random.default_rng(0xA1)
    cfgs = [(16, 64, 64, 16, 16, 64), (64, 32, 32, 32, 32, 32), (64, 64, 64, 32, 64, 64),
            (128, 128, 64, 64, 32, 32), (256, 128, 128, 64, 64, 32)]
    for it in range(12):
        m, k, n = (int(v) for v in rng.integers(1, 200, 3))
        a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        cfg = cfgs[it % len(cfgs)]
        assert np.array_equal(oracle.atmm_multiply(a, b, cfg), reference.atmm_multiply(a, b, cfg))


def test_run_bypass_live_cfg1_shape(oracle, reference):
    """BASELINE configs[0] (hidden 4096, rank 16, 4 adapters, 64 tokens): oracle == reference bits."""
    d = 4096
    adapters = {}
    for a in range(4):
        dn, u = oracle.adapter_random(1000 + a, 1, d, 16)
        adapters[a] = (dn[0], u[0])
    x = oracle.random_matrix(oracle.rng(7), 64, d)
    assignment = np.asarray(oracle.seeded_shuffle(oracle.rng(3), np.repeat(np.arange(4), 16)), np.int32)
    ctx = reference.ctx(d, adapters)
    assert np.array_equal(oracle.run_bypass(x, assignment, adapters), ctx.run_bypass(x, assignment))


# ------------------------------------------------------- stack forward ---


def _fwd_gold_adapters(gold):
    return {a: (gold[f"fwd_down_{a}"], gold[f"fwd_up_{a}"]) for a in (1, 2)}


@pytest.mark.parametrize("mode", ["unmerged", "mixture", "merged"])
def test_forward_matches_reference_golden(oracle, gold, mode):
    """orc_forward_f64 restates forward_unmerged / forward_mixture /
    forward_merged (model.hpp:192-328); pinned to the reference's own outputs
    in the mode-equivalence setting of verify.hpp:63-100."""
    ads = _fwd_gold_adapters(gold)
    w = gold["fwd_w"] if mode == "unmerged" else gold["fwd_w_merged"]
    got = oracle.forward_f64(gold["fwd_x"], w, mode, gold["fwd_assignment"], ads, merged_id=1, round_act=False)
    want = gold[f"fwd_{mode}"]
    assert np.max(np.abs(got - want)) <= 1e-4 * max(1.0, float(np.max(np.abs(want))))


def test_forward_mode_equivalence_golden(gold):
    """verify.hpp:89-100: mixture rows of the merged adapter equal the merged
    forward, every other row equals the unmerged forward."""
    a = gold["fwd_assignment"]
    tol = 1e-4 * max(1.0, float(np.max(np.abs(gold["fwd_unmerged"]))))
    for row in range(a.size):
        other = gold["fwd_merged"] if a[row] == 1 else gold["fwd_unmerged"]
        assert np.max(np.abs(gold["fwd_mixture"][row] - other[row])) <= tol


@pytest.mark.parametrize("seed", [1, 2])
def test_forward_live(oracle, reference, seed):
    rng = np.random.default_rng(seed)
    L, d, n = 2, 96, 13
    w = oracle.model_random(seed, L, d)
    ads = {}
    for a, r in {3: 8, 4: 24, 9: 16}.items():
        ads[a] = oracle.adapter_random(100 * seed + a, L, d, r)
    x = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    assignment = rng.choice([3, 4, 9], n).astype(np.int32)
    want, _ = reference.forward(x, w, "unmerged", assignment, ads)
    got = oracle.forward_f64(x, w, "unmerged", assignment, ads, round_act=False)
    assert np.max(np.abs(got - want)) <= 1e-4
    want, wm = reference.forward(x, w, "mixture", assignment, ads, merged_id=4)
    got = oracle.forward_f64(x, wm, "mixture", assignment, ads, merged_id=4, round_act=False)
    assert np.max(np.abs(got - want)) <= 1e-4
