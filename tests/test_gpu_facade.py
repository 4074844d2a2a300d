"""The C++ drop-in facade (include/uot/cuda.hpp) run against the reference in
C++: tests/cpp/test_facade.cpp, built into oracle/_ref/test_facade by
`make -C oracle facade`, and the reference's OWN acceptance gate
(proj/tests/acceptance.cpp, 11 criteria) with its solver calls routed to
uot::cuda (`make -C oracle acceptance_gpu`). Both need /root/reference at build
time only."""
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


ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_gpu")


def test_reference_acceptance_gate_on_the_gpu_backend(gpu):
    # c01 solver agreement (baseline / fused / fused W=4 / tiled / distributed(3), 20 fp64
    # problems, <= 1e-10, < 10 s), c08 balanced convergence, c09 fused faster than baseline,
    # c10 distributed invariants (CommStats, P=1 == serial bitwise) run on the GPU; the
    # CPU-model criteria (intensity, roofline, traffic, cache, traces) stay the reference's
    if not os.path.exists(ACC):
        pytest.skip("oracle/_ref/acceptance_gpu not built (needs /root/reference at build time)")
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 11
