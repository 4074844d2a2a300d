"""The C++ drop-in facade (include/uot/cuda.hpp) run against the reference in
C++: tests/cpp/test_facade.cpp, built into oracle/_ref/test_facade by
`make -C oracle facade` (needs /root/reference at build time only)."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "test_facade")


def test_cpp_facade_suite(gpu):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_facade not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
