"""The B200 tiling search (atmm.hpp:188-355 re-read for the fused bypass).

Host-only: the selection half of tiling_search (per-shape argmin, ties to the
lexicographically smallest candidate, failed shapes omitted and reported, the
most frequent winner as default -- atmm.hpp:293-329), the default grid and
candidates, the JSON round trip with the "sm100" / "default_sm100" launch
extension (read back identically by the reference's own TilingTable::load).
GPU: benchmark_config's trials rule, grid_bench_ns shape, and a small search
whose table resolves every grid shape to its measured argmin."""
import numpy as np
import pytest

MAX = np.iinfo(np.int64).max


def test_table_from_scores_argmin_ties_failures_default(atmm):
    shapes = [(32, 4096, 16, 4096, 16), (64, 4096, 16, 4096, 16), (128, 4096, 64, 4096, 8),
              (256, 4096, 64, 4096, 4), (512, 5120, 32, 5120, 4)]
    launches = [(32, 8, 128, 0, 0), (16, 8, 128, 0, 0), (64, 4, 128, 0, 1), (128, 8, 256, 0, 0)]
    scores = [[100, 90, 95, 99],      # argmin -> launch 1
              [50, 50, 60, 70],       # tie 0/1 -> lexicographically smaller (16,...) = launch 1
              [MAX, 30, 20, 40],      # argmin -> launch 2 (launch 0 failed)
              [10, 11, 12, 9],        # argmin -> launch 3
              [MAX, MAX, MAX, MAX]]   # all failed: omitted
    fails = []
    t = atmm.table_from_scores(shapes, launches, scores, fails)
    assert len(t) == 4
    assert t.resolve_launch(32, 4096, 16, 4096) == (16, 8, 128, 0, 0)
    assert t.resolve_launch(64, 4096, 16, 4096) == (16, 8, 128, 0, 0)
    assert t.resolve_launch(128, 4096, 64, 4096) == (64, 4, 128, 0, 1)
    assert t.resolve_launch(256, 4096, 64, 4096) == (128, 8, 256, 0, 0)
    assert len(fails) == 1 and "omitted" in fails[0]
    # the most frequent winner (launch 1, two wins) is the default for misses
    assert t.resolve_launch(1000, 777, 3, 777) == (16, 8, 128, 0, 0)
    # nearest same-(k, n) bucket within 32 (tiling.hpp:181-199)
    assert t.resolve_launch(90, 4096, 16, 4096) == (16, 8, 128, 0, 0)


def test_table_from_scores_duplicate_key_prefers_larger_batch(atmm):
    launches = [(32, 8, 128, 0, 0), (64, 8, 128, 0, 0)]
    # same key (m_bucket 64, 4096, 16): the 16 x 64-row batch wins although slower
    shapes = [(33, 4096, 16, 4096, 8), (64, 4096, 16, 4096, 16)]
    t = atmm.table_from_scores(shapes, launches, [[10, 20], [30, 25]])
    assert len(t) == 1 and t.resolve_launch(64, 4096, 16, 4096) == (64, 8, 128, 0, 0)
    t = atmm.table_from_scores(shapes[::-1], launches, [[30, 25], [10, 20]])
    assert t.resolve_launch(64, 4096, 16, 4096) == (64, 8, 128, 0, 0)
    # equal batches: the faster measurement wins (atmm.hpp:311-315)
    shapes = [(64, 4096, 16, 4096, 8), (64, 4096, 16, 4096, 8)]
    t = atmm.table_from_scores(shapes, launches, [[10, 20], [30, 5]])
    assert t.resolve_launch(64, 4096, 16, 4096) == (64, 8, 128, 0, 0)


def test_default_grid_and_candidates(atmm):
    g = atmm.default_shape_grid(4096)
    assert len(g) == 8 * 5
    assert {s[2] for s in g} == {8, 16, 32, 64, 128}
    assert {s[0] for s in g} == {8, 16, 32, 64, 96, 128, 256, 512}
    assert all(s[1] == s[3] == 4096 and 4 <= s[4] <= 64 for s in g)
    assert atmm.default_shape_grid(5120, ranks=[64]) == [s for s in atmm.default_shape_grid(5120) if s[2] == 64]
    c = atmm.default_launch_candidates()
    assert len(c) == len(set(c)) >= 12
    assert all(len(x) == 5 for x in c)


def test_search_table_json_round_trip_reference_loadable(atmm, tmp_path, reference):
    import ctypes

    shapes = [(32, 4096, 16, 4096, 16), (256, 4096, 64, 4096, 4)]
    launches = [(32, 16, 128, 0, 0), (128, 8, 256, 0, 2)]
    t = atmm.table_from_scores(shapes, launches, [[5, 6], [9, 8]])
    p = str(tmp_path / "t.json")
    t.save(p)
    back = atmm.TilingTable.load(p)
    for m, k, n in [(32, 4096, 16), (256, 4096, 64), (7, 7, 7)]:
        assert back.resolve_launch(m, k, n, k) == t.resolve_launch(m, k, n, k)
        out = np.zeros(6, np.int32)
        st = reference.L.ref_table_load_lookup(p.encode(), m, k, n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        assert st == 0 and tuple(out) == back.lookup(m, k, n)
    assert back.resolve_launch(256, 4096, 64, 4096)[4] == 2  # the forced path survives the round trip


def test_packaged_table_loads_and_covers_bench_configs(atmm):
    import os

    p = os.path.join(os.path.dirname(atmm.__file__), "tables", "b200_tiling_table.json")
    if not os.path.exists(p):
        pytest.skip("no packaged table yet")
    t = atmm.TilingTable.load(p)
    assert len(t) > 0
    for m, d, r in [(16, 4096, 16), (32, 4096, 16), (128, 5120, 64)]:
        assert t.find_entry(m, d, r) is not None


@pytest.mark.gpu
def test_benchmark_and_small_search(gpu, atmm):
    shape = (32, 1024, 16, 1024, 8)
    with pytest.raises(atmm.ConfigError):
        atmm.benchmark_launch(shape, (32, 4, 128, 0, 0), trials=2)  # test_atmm.cpp:127-129
    ns = atmm.benchmark_launch(shape, (32, 4, 128, 0, 0), trials=3)
    assert 0 < ns < 10_000_000
    shapes = [shape, (128, 1024, 32, 1024, 4)]
    launches = [(32, 4, 128, 0, 0), (16, 8, 128, 0, 0), (128, 2, 128, 0, 2)]
    scores = atmm.grid_bench_ns(shapes, launches, trials=3, rounds=2)
    assert scores.shape == (2, 3) and np.all(scores > 0) and np.all(scores < MAX)
    fails = []
    t = atmm.tiling_search(shapes, launches, trials=3, failures=fails)
    assert len(t) == 2 and not fails
    for sh in shapes:
        got = t.resolve_launch(sh[0], sh[1], sh[2], sh[3])
        assert got in [tuple(l) for l in launches]
