"""Execution modes of one iterate() call give the same answers.

* streaming: one sweep launch + one finalize launch per iteration (sweep.cuh,
  finalize.cuh) — any shape;
* resident: the whole call is ONE cooperative launch with the matrix in shared
  memory and two grid barriers per iteration (resident.cuh) — small shapes
  (uot_set_resident(ctx, 0) forces streaming);
* the two row-batch schedules of the streaming sweep: fixed row blocks (the
  default, bit-reproducible) and the dynamic batch counter.

Each mode is checked against the CPU oracle (fused_solve, fused.hpp:259-291)
and the modes against each other, including the early exit and the
degenerate-sum paths the reference defines (fused.hpp:273-281, scaling.cpp:15-22).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import KNEVER
from test_gpu_parity import assert_parity

pytestmark = pytest.mark.gpu


def run(uot, a, rpd, cpd, er, ep, k, tol=KNEVER, resident=True, chunks=None, deterministic=True):
    with uot.Session(a.shape[0], a.shape[1]) as s:
        s.set_resident(resident)
        s.set_deterministic(deterministic)
        lay = s.layout
        s.set_problem(uot.Problem(a, rpd, cpd, er, ep))
        s.init_col_sums()
        done = 0
        for c in (chunks or [k]):
            it, err, conv = s.iterate(c, tol)
            done += it
            if conv:
                break
        return s.plan(), s.factors(), s.col_sums(), done, err, conv, lay


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 40), (2000, 513, 30), (16, 16, 25), (3, 7, 9), (300, 4096, 12)])
def test_resident_matches_streaming_and_oracle(gpu, orc, m, n, k):
    a, rpd, cpd = orc.gen_problem(42, m, n)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 4)
    res = run(gpu, a, rpd, cpd, 1.0, 0.1, k)
    stream = run(gpu, a, rpd, cpd, 1.0, 0.1, k, resident=False)
    assert res[6]["resident"] == 1 and stream[6]["resident"] == 0
    for plan, f, cs, it, err, conv, lay in (res, stream):
        assert it == k
        assert_parity(plan, ref.plan, rpd, cpd, f"{m}x{n} resident={lay['resident']}")
        np.testing.assert_allclose(f.alpha, ref.alpha, rtol=1e-12)
        np.testing.assert_allclose(f.beta, ref.beta, rtol=1e-12)
        np.testing.assert_allclose(cs, ref.col_sums, rtol=1e-12)
        assert abs(err - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)


def test_resident_is_resumable_across_calls(gpu, orc):
    # k iterations in one launch == the same k split over several calls
    a, rpd, cpd = orc.gen_problem(8, 500, 777)
    one = run(gpu, a, rpd, cpd, 1.0, 0.1, 12)
    split = run(gpu, a, rpd, cpd, 1.0, 0.1, 12, chunks=[5, 1, 6])
    assert one[6]["resident"] == 1
    assert np.array_equal(one[0], split[0]) and split[3] == 12
    np.testing.assert_array_equal(one[1].beta, split[1].beta)


def test_resident_stops_at_the_reference_iteration(gpu, orc):
    a, rpd, cpd = orc.gen_problem(37, 24, 24)
    cpd = cpd * (rpd.sum() / cpd.sum())
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.0, 1e-6, 10000, 1)
    r = run(gpu, a, rpd, cpd, 1.0, 0.0, 10000, tol=1e-6)
    assert r[6]["resident"] == 1 and ref.converged and r[5]
    assert r[3] == ref.iterations
    assert_parity(r[0], ref.plan, rpd, cpd, "resident converged")


def test_resident_degenerate_column_sums_raise(gpu, orc):
    a, rpd, cpd = orc.gen_problem(38, 4, 4)
    with gpu.Session(4, 4) as s:
        assert s.layout["resident"] == 1
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 1.0))
        s.set_col_sums(np.zeros(4))
        with pytest.raises(gpu.DegenerateSum):
            s.iterate(3, KNEVER)
        np.testing.assert_array_equal(s.plan(), a)


@pytest.mark.parametrize("m,n,k", [(3000, 32768, 4), (20000, 4096, 5), (4099, 8192, 4)])
def test_batch_schedules(gpu, orc, m, n, k):
    """The deterministic schedule (default: fixed row blocks) and dynamic batches
    (a device counter hands out row batches, uot_set_deterministic(0)) both meet
    the parity bar; the deterministic one reproduces itself bit for bit."""
    a, rpd, cpd = orc.gen_problem(11, m, n)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 4)
    out = {}
    for name, det in (("det1", True), ("det2", True), ("dyn", False)):
        with gpu.Session(m, n) as s:
            s.set_deterministic(det)
            assert s.layout["dynamic"] == (0 if det else 1)
            s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.1))
            s.init_col_sums()
            it, err, conv = s.iterate(k, KNEVER)
            assert it == k
            out[name] = (s.plan(), s.factors())
        assert_parity(out[name][0], ref.plan, rpd, cpd, f"{m}x{n} {name}")
        np.testing.assert_allclose(out[name][1].alpha, ref.alpha, rtol=1e-10)
    assert np.array_equal(out["det1"][0], out["det2"][0])
    np.testing.assert_array_equal(out["det1"][1].alpha, out["det2"][1].alpha)
