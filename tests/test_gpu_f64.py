"""Problem<double> (Dtype::f64, matrix.hpp:13) on the device path.

With T = double the reference's row pass (fused.hpp:128-140) multiplies and
adds in f64 with no narrowing, so the sweep stores plain f64 products; the
oracle's f64 solver (itself pinned to the reference, tests/test_oracle.py)
is the check. Plans agree to the f64 summation order (~1e-15), far inside the
1e-5 bar.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, KNEVER
from test_gpu_parity import assert_parity

pytestmark = pytest.mark.gpu


def solve64(uot, a, rpd, cpd, er, ep, k, tol=KNEVER):
    with uot.Session(a.shape[0], a.shape[1], dtype=np.float64) as s:
        assert s.layout["dtype"] == 2
        s.set_problem(uot.Problem(a, rpd, cpd, er, ep))
        s.init_col_sums()
        it, err, conv = s.iterate(k, tol)
        return s.plan(), s.factors(), s.col_sums(), it, err, conv, s.layout


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 40), (300, 20000, 8), (64, 32768, 6), (2000, 513, 20),
                                   (5, 7, 9), (4096, 4096, 6), (777, 4097, 7)])
def test_f64_matches_oracle(gpu, orc, m, n, k):
    a, rpd, cpd = orc.gen_problem(42, m, n, dtype=np.float64)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 4)
    plan, f, cs, it, err, conv, lay = solve64(gpu, a, rpd, cpd, 1.0, 0.1, k)
    assert plan.dtype == np.float64 and it == k
    rel = assert_parity(plan, ref.plan, rpd, cpd, f"f64 {m}x{n}")
    assert rel <= 1e-12, f"f64 plan differs by {rel:.3e}"
    np.testing.assert_allclose(f.alpha, ref.alpha, rtol=1e-12)
    np.testing.assert_allclose(f.beta, ref.beta, rtol=1e-12)
    np.testing.assert_allclose(cs, ref.col_sums, rtol=1e-12)
    assert abs(err - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)


def test_f64_device_generator_is_bit_exact(gpu, orc):
    m, n = 333, 5000
    a, rpd, cpd = orc.gen_problem(7, m, n, dtype=np.float64)
    with gpu.Session(m, n, dtype=np.float64) as s:
        s.generate_problem(7, 1.0, 0.5)
        assert np.array_equal(s.plan(), a)
    host = gpu.gen_problem_t(7, m, n, dtype=np.float64)
    assert np.array_equal(host.a, a) and np.array_equal(host.rpd, rpd) and np.array_equal(host.cpd, cpd)


def test_f64_converges_at_the_reference_iteration(gpu, orc):
    a, rpd, cpd = orc.gen_problem(37, 300, 9000, dtype=np.float64)
    cpd = cpd * (rpd.sum() / cpd.sum())
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.0, 1e-9, 10000, 1)
    plan, f, cs, it, err, conv, lay = solve64(gpu, a, rpd, cpd, 1.0, 0.0, 10000, tol=1e-9)
    assert ref.converged and conv and it == ref.iterations
    assert_parity(plan, ref.plan, rpd, cpd, "f64 converged")


def test_f64_fused_solve_keeps_double(gpu, orc):
    a, rpd, cpd = orc.gen_problem(3, 40, 60, dtype=np.float64)
    r = gpu.fused_solve(gpu.Problem(a, rpd, cpd, 1.0, 0.2), KNEVER, 5)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.2, KNEVER, 5, 1)
    assert r.plan.dtype == np.float64
    assert_parity(r.plan, ref.plan, rpd, cpd, "fused_solve f64")


def test_f64_file_round_trip_and_dtype_checks(gpu, tmp_path):
    src = os.path.join(GOLDEN, "io_2x2_f64.uotp")
    with gpu.Session(2, 2, dtype=np.float64) as s:
        s.load_problem_file(src)
        s.save_problem_file(tmp_path / "back.uotp")
        with pytest.raises(gpu.InvalidParameter):  # a Problem<float> container into a double session
            s.load_problem_file(os.path.join(GOLDEN, "io_6x4_er2.5_ep0.5.uotp"))
    assert (tmp_path / "back.uotp").read_bytes() == open(src, "rb").read()
    with gpu.Session(2, 2) as s:
        with pytest.raises(gpu.InvalidParameter):  # and the other way round
            s.load_problem_file(src)
