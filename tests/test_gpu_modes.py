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
    """The three row-batch schedules (uot_set_schedule) meet the parity bar; the
    two static ones reproduce themselves bit for bit."""
    a, rpd, cpd = orc.gen_problem(11, m, n)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 4)
    out = {}
    for name, mode in (("cw1", "class_weighted"), ("cw2", "class_weighted"), ("u1", "uniform"),
                       ("u2", "uniform"), ("dyn", "dynamic")):
        with gpu.Session(m, n) as s:
            s.set_schedule(mode)
            assert s.layout["schedule"] == gpu.Session.SCHEDULES[mode]
            assert s.layout["dynamic"] == (1 if mode == "dynamic" else 0)
            s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.1))
            s.init_col_sums()
            it, err, conv = s.iterate(k, KNEVER)
            assert it == k
            out[name] = (s.plan(), s.factors(), s.col_sums())
        assert_parity(out[name][0], ref.plan, rpd, cpd, f"{m}x{n} {name}")
        np.testing.assert_allclose(out[name][1].alpha, ref.alpha, rtol=1e-10)
    for x, y in (("cw1", "cw2"), ("u1", "u2")):
        assert np.array_equal(out[x][0], out[y][0])
        np.testing.assert_array_equal(out[x][1].alpha, out[y][1].alpha)
        np.testing.assert_array_equal(out[x][2], out[y][2])


@pytest.mark.slow
def test_default_schedule_is_bit_reproducible_at_scale(gpu, orc):
    """Two default runs (separate sessions) of a problem far past the 64 MiB
    threshold give identical bits: plan, factors, carried column sums and error
    (the reference's promise, fused.hpp:193-196, 242-248)."""
    m, n, k = 16384, 20000, 6  # 1.2 GiB, G = 3 ... and one CTA per SM where the grid allows
    runs = []
    for _ in range(2):
        with gpu.Session(m, n) as s:
            assert s.layout["schedule"] == 0 and s.layout["dynamic"] == 0
            s.generate_problem(42, 1.0, 0.1)
            s.init_col_sums()
            it, err, conv = s.iterate(k, KNEVER)
            f = s.factors()
            runs.append((s.plan(), f.alpha, f.beta, s.col_sums(), err))
    for x, y in zip(runs[0], runs[1]):
        assert np.array_equal(np.asarray(x), np.asarray(y))
    for (m, n) in [(8192, 32768), (65536, 4096)]:  # G = 4 and G = 1 with one CTA per SM
        runs = []
        for _ in range(2):
            with gpu.Session(m, n) as s:
                s.generate_problem(7, 1.0, 0.1)
                s.init_col_sums()
                s.iterate(4, KNEVER)
                runs.append((s.plan(), s.factors().beta, s.layout["sm_classes"]))
        assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
        assert runs[0][2] == runs[1][2]


def test_sm_classes_and_weighted_blocks(gpu):
    """The probe's classes drive the schedule: every CTA's SM is recorded, the
    groups' weights are per class, and a class-weighted sweep streams every row
    exactly once (batch counts add up to the rows)."""
    cls, ms = gpu.sm_classes(0)
    assert cls.size == ms.size and cls.size >= 1
    m, n = 20000, 4096
    with gpu.Session(m, n) as s:
        s.generate_problem(3, 1.0, 0.1)
        s.init_col_sums()
        s.iterate(2, KNEVER)
        smid, nb, w = s.schedule_stats()
        lay = s.layout
    assert len(set(smid.tolist())) == smid.size  # one CTA per SM
    rows_per_batch = lay["rows_per_step"]
    assert nb.sum() * rows_per_batch >= m and (nb.sum() - smid.size) * rows_per_batch < m
    if lay["sm_classes"] > 0:
        assert len(set(w.tolist())) <= lay["sm_classes"] + 1
