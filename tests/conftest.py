import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device; run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (reference headers were not available at build time)")
    return Reference()


@pytest.fixture(scope="session")
def atmm():
    import paper_2411_00915_b200 as m

    return m


@pytest.fixture(scope="session")
def gpu(atmm):
    # GPU tests never silently pass on a CPU host: no device is a failure.
    n = atmm.device_count()
    assert n > 0, "no sm_100 device visible (the -m gpu suite must run on a B200)"
    import torch

    torch.cuda.init()
    return 0


def tol_for(ref) -> float:
    """North-star tolerance (BASELINE.json): 1e-2 * max(1, max|ref|), bf16 in / fp32 acc."""
    return 1e-2 * max(1.0, float(np.max(np.abs(ref))) if np.size(ref) else 0.0)


PATH_CODES = {"auto": 0, "a2a": 1, "split": 2, "fused": 3, "stream": 4}


def path_table(atmm, assignment, ranks, d_in, d_out, path):
    """A tiling table whose entry for every segment of this batch is the
    heuristic launch with the kernel path forced (ATMM_PATH_*), i.e. the
    automatic plan except for the kernel choice.  None for "auto"."""
    if path == "auto":
        return None
    t = atmm.TilingTable()
    a = np.asarray(assignment)
    for aid in np.unique(a):
        m = int(np.count_nonzero(a == aid))
        r = int(ranks[int(aid)])
        launch = list(atmm.heuristic_launch(m, d_in, r, d_out))
        launch[4] = PATH_CODES[path]
        t.insert(atmm.m_bucket_of(m), d_in, r, (128, 128, 256, 128, 16, 64), 1, sm100=launch)
    return t
