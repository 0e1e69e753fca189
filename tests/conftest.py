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
