"""Shared fixtures. `-m gpu` tests need a B200 and the built extension; the rest
run on CPU (oracle vs the reference, the C ABI surface, host logic, gloo)."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
KNEVER = 1e-300  # positive but unreachable: fixed-length runs (acceptance.cpp:26)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a extension")
    config.addinivalue_line("markers", "slow: large problem sizes")


def er_ep(fi):
    """oracle.hpp:61-67 — er fixed at 1, ep chosen so that er/(er+ep) == fi."""
    return 1.0, (1.0 - fi) / fi


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref (the reference compiled from /root/reference) is not available")
    return oracle.RefOracle()


@pytest.fixture(scope="session")
def small_golden():
    data = np.load(os.path.join(GOLDEN, "small.npz"))
    with open(os.path.join(GOLDEN, "small.json")) as f:
        meta = json.load(f)
    return data, meta


@pytest.fixture(scope="session")
def big_golden():
    path = os.path.join(GOLDEN, "big.npz")
    if not os.path.exists(path):
        pytest.skip("tests/golden/big.npz not generated")
    with open(os.path.join(GOLDEN, "big.json")) as f:
        meta = json.load(f)
    return np.load(path), meta


def cuda_ok() -> bool:
    try:
        import ctypes
        n = ctypes.c_int(0)
        lib = ctypes.CDLL("libcuda.so.1")
        if lib.cuInit(0) != 0:
            return False
        lib.cuDeviceGetCount(ctypes.byref(n))
        return n.value > 0
    except OSError:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not cuda_ok():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2412_11079_b200 import uot
    uot.lib()
    return uot
