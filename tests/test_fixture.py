"""Reference fixture formats (matrix.hpp:183-218, model_io.hpp:25-114) on CPU.

Files written by the reference itself (oracle/_ref: save_matrix,
save_model_fixture) are read by our loader bit-exactly, ours are byte-identical
to the reference's, and the error behaviour matches (IoError on truncated
files and scalar-width mismatch).
"""
import json
import os

import numpy as np
import pytest


def _ref_save_matrix(reference, path, m):
    import ctypes

    a = np.ascontiguousarray(m, np.float32)
    st = reference.L.ref_save_matrix(str(path).encode(), a.shape[0], a.shape[1],
                                     a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    assert st == 0


def test_matrix_roundtrip_and_reference_bytes(atmm, reference, tmp_path):
    rng = np.random.default_rng(3)
    for shape in [(1, 1), (7, 13), (64, 16), (0, 5)]:
        m = rng.uniform(-1, 1, shape).astype(np.float32)
        ours, theirs = tmp_path / f"o{shape}.bin", tmp_path / f"r{shape}.bin"
        atmm.save_matrix(ours, m)
        _ref_save_matrix(reference, theirs, m)
        assert ours.read_bytes() == theirs.read_bytes()
        back = atmm.load_matrix(theirs)
        assert back.shape == shape and np.array_equal(back, m)


def test_matrix_errors(atmm, tmp_path):
    m = np.arange(12, dtype=np.float32).reshape(3, 4)
    p = tmp_path / "m.bin"
    atmm.save_matrix(p, m)
    raw = p.read_bytes()
    (tmp_path / "short.bin").write_bytes(raw[:-4])
    with pytest.raises(atmm.IoError, match="truncated payload"):
        atmm.load_matrix(tmp_path / "short.bin")
    (tmp_path / "hdr.bin").write_bytes(raw[:6])
    with pytest.raises(atmm.IoError, match="truncated header"):
        atmm.load_matrix(tmp_path / "hdr.bin")
    bad = bytearray(raw)
    bad[8] = 8  # scalar width 8 (double) in a float file
    (tmp_path / "w.bin").write_bytes(bytes(bad))
    with pytest.raises(atmm.IoError, match="scalar width mismatch"):
        atmm.load_matrix(tmp_path / "w.bin")
    with pytest.raises(atmm.IoError, match="cannot open"):
        atmm.load_matrix(tmp_path / "missing.bin")


def write_reference_fixture(reference, directory, L, d, adapters, seed=5):
    """save_model_fixture of the reference with the given {id: (down[L], up[L])}."""
    import ctypes

    ids = np.asarray(sorted(adapters), np.int32)
    ranks = np.asarray([adapters[i][0].shape[2] for i in ids], np.int64)
    flat = np.concatenate([np.concatenate([adapters[i][0].reshape(-1), adapters[i][1].reshape(-1)]) for i in ids])
    flat = np.ascontiguousarray(flat, np.float32)
    st = reference.L.ref_save_fixture(str(directory).encode(), L, d, 16, seed, ids.size,
                                      ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                      ranks.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                      flat.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    assert st == 0


def test_reference_fixture_manifest_and_files(atmm, reference, tmp_path):
    L, d = 3, 32
    rng = np.random.default_rng(9)
    adapters = {}
    for aid, r in [(4, 8), (11, 16)]:
        adapters[aid] = (rng.uniform(-1, 1, (L, d, r)).astype(np.float32), rng.uniform(-1, 1, (L, r, d)).astype(np.float32))
    write_reference_fixture(reference, tmp_path, L, d, adapters)
    info = atmm.fixture_info(tmp_path)
    assert info == {"num_layers": L, "hidden_dim": d, "adapters": {4: 8, 11: 16}}
    man = json.loads((tmp_path / "manifest.json").read_text())
    for a in man["adapters"]:
        for l, (fd, fu) in enumerate(zip(a["down"], a["up"])):
            assert np.array_equal(atmm.load_matrix(tmp_path / fd), adapters[a["id"]][0][l])
            assert np.array_equal(atmm.load_matrix(tmp_path / fu), adapters[a["id"]][1][l])
    # a manifest listing the wrong layer count is an IoError (model_io.hpp:84-86 style)
    man["adapters"][0]["down"] = man["adapters"][0]["down"][:1]
    (tmp_path / "manifest.json").write_text(json.dumps(man))
    with pytest.raises(atmm.IoError, match="wrong layer count"):
        atmm.fixture_info(tmp_path)
    (tmp_path / "manifest.json").write_text("{not json")
    with pytest.raises(atmm.IoError, match="bad manifest"):
        atmm.fixture_info(tmp_path)
    os.remove(tmp_path / "manifest.json")
    with pytest.raises(atmm.IoError, match="cannot read manifest"):
        atmm.fixture_info(tmp_path)
