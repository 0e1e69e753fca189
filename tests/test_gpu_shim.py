"""GPU: the header-only C++ shim (include/loraserve_b200.hpp) end to end on
the device -- run_bypass / atmm_multiply / delta_w KATs and exception types,
written like the reference's Catch2 cases (tests/cpp/shim_test.cpp)."""
import subprocess

import pytest

from test_host import _build_shim

pytestmark = pytest.mark.gpu


def test_cpp_shim_gpu_cases(gpu, tmp_path):
    exe = _build_shim(tmp_path)
    out = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
