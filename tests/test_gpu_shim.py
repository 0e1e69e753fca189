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


def test_reference_acceptance_criteria_through_compat_header(gpu, tmp_path):
    """acceptance.cpp criteria 1-4 + the mode contract through
    include/loraserve_compat.hpp (reference signatures) on the B200."""
    from test_host import _build_acceptance

    exe = _build_acceptance(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 5
