"""Builds libatmm_b200.so in-tree for sm_100a (and the oracle checkers).

    python -m paper_2411_00915_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_library(verbose: bool = False) -> str:
    csrc = os.path.join(ROOT, "paper_2411_00915_b200", "csrc")
    out = subprocess.run(["make", "-C", csrc, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        sys.stderr.write(out.stdout + out.stderr)
        raise RuntimeError("building libatmm_b200.so failed")
    if verbose:
        sys.stdout.write(out.stdout)
    return os.path.join(ROOT, "paper_2411_00915_b200", "libatmm_b200.so")


def build_oracle(verbose: bool = False) -> None:
    """Test infrastructure: oracle/_build (C restatement) and, when the
    reference is mounted, oracle/_ref (the reference compiled in place)."""
    out = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], capture_output=True, text=True)
    if out.returncode != 0:
        sys.stderr.write(out.stdout + out.stderr)
        raise RuntimeError("building the oracle failed")
    if verbose:
        sys.stdout.write(out.stdout)


if __name__ == "__main__":
    build_library(verbose=True)
    build_oracle(verbose=True)
