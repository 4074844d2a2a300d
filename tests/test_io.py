"""Problem files (.uotp, problem_io.cpp:13-141) — host side, no GPU.

The golden containers in tests/golden/*.uotp were written by the unmodified
reference (tests/golden/make_uotp.py). The checks mirror test_io.cpp: header
layout, bit-exact round trips, and the malformed-container cases of
test_io.cpp:172-194 raising IoError.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN

CASES = [("io_6x4_er2.5_ep0.5.uotp", 5, 6, 4, 2.5, 0.5), ("io_64x100.uotp", 11, 64, 100, 1.0, 0.1),
         ("io_37x1000.uotp", 3, 37, 1000, 1.0, 0.25)]


@pytest.fixture(scope="module")
def uot():
    from paper_2412_11079_b200 import uot
    uot.lib()
    return uot


@pytest.mark.parametrize("name,seed,m,n,er,ep", CASES)
def test_reference_containers_parse(uot, orc, name, seed, m, n, er, ep):
    path = os.path.join(GOLDEN, name)
    assert uot.problem_file_info(path) == {"m": m, "n": n, "dtype": "f32", "er": er, "ep": ep}
    p = uot.read_problem(path)
    a, rpd, cpd = orc.gen_problem(seed, m, n)  # the generator the reference wrote them from
    assert np.array_equal(p.a, a) and np.array_equal(p.rpd, rpd) and np.array_equal(p.cpd, cpd)
    assert (p.er, p.ep) == (er, ep)


@pytest.mark.parametrize("name,seed,m,n,er,ep", CASES)
def test_write_is_byte_identical_to_the_reference(uot, orc, tmp_path, name, seed, m, n, er, ep):
    a, rpd, cpd = orc.gen_problem(seed, m, n)
    out = tmp_path / "mine.uotp"
    uot.write_problem(out, uot.Problem(a, rpd, cpd, er, ep))
    assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read()


def test_f64_container(uot, orc):
    # a Problem<double> container written by the reference (make_uotp.py: the
    # seed-5 2x2 fp32 draw widened to double)
    path = os.path.join(GOLDEN, "io_2x2_f64.uotp")
    info = uot.problem_file_info(path)
    assert info["dtype"] == "f64" and (info["m"], info["n"]) == (2, 2)
    p = uot.read_problem(path)
    a, rpd, cpd = orc.gen_problem(5, 2, 2)
    assert p.a.dtype == np.float64 and np.array_equal(p.a, a.astype(np.float64))
    assert np.array_equal(p.rpd, rpd) and np.array_equal(p.cpd, cpd) and p.ep == 0.25


def test_f64_write_is_byte_identical(uot, orc, tmp_path):
    a, rpd, cpd = orc.gen_problem(5, 2, 2)
    out = tmp_path / "f64.uotp"
    uot.write_problem(out, uot.Problem(a.astype(np.float64), rpd, cpd, 1.0, 0.25))
    assert out.read_bytes() == open(os.path.join(GOLDEN, "io_2x2_f64.uotp"), "rb").read()


def test_malformed_containers_raise_ioerror(uot, tmp_path):
    # test_io.cpp:172-194
    good = open(os.path.join(GOLDEN, "io_2x2_f64.uotp"), "rb").read()
    mutations = [
        lambda b: b[:0] + b"X" + b[1:],                   # magic
        lambda b: b[:4] + bytes([2]) + b[5:],             # unsupported version
        lambda b: b[:6] + bytes([3]) + b[7:],             # unknown dtype code
        lambda b: b[:-1],                                  # truncated payload
        lambda b: b + b"\0",                               # trailing garbage
        lambda b: b[:8] + bytes([0]) + b[9:],             # M = 0
        lambda b: b[:12],                                  # not even a header
    ]
    for k, mutate in enumerate(mutations):
        p = tmp_path / f"bad{k}.uotp"
        p.write_bytes(mutate(good))
        with pytest.raises(uot.IoError):
            uot.problem_file_info(p)
    with pytest.raises(uot.IoError):
        uot.problem_file_info("/nonexistent/uot/path.uotp")


def test_reference_reads_what_we_write(uot, ref, tmp_path, orc):
    a, rpd, cpd = orc.gen_problem(21, 9, 13)
    out = tmp_path / "w.uotp"
    uot.write_problem(out, uot.Problem(a, rpd, cpd, 1.5, 0.125))
    dt, er, ep, ra, rr, rc = ref.read_problem(out)
    assert dt == "f32" and (er, ep) == (1.5, 0.125)
    assert np.array_equal(ra, a) and np.array_equal(rr, rpd) and np.array_equal(rc, cpd)
