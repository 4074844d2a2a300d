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
    with uot.Session(a.shape[0], a.shape[1], dtype=a.dtype) as s:
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
    two static ones reproduce themselves bit for bit (weighted: for the same
    weights, in another session)."""
    a, rpd, cpd = orc.gen_problem(11, m, n)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 4)
    out = {}
    weights = None
    for name in ("u1", "u2", "w1", "w2", "dyn"):
        with gpu.Session(m, n) as s:
            s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.1))
            s.init_col_sums()
            if name == "w1":
                weights = s.calibrate_schedule(3)  # the plan is untouched by the scratch run
                assert np.array_equal(s.plan(), a)
            elif name == "w2":
                s.set_group_weights(weights)
            elif name == "dyn":
                s.set_schedule("dynamic")
            mode = {"u": "uniform", "w": "weighted", "d": "dynamic"}[name[0]]
            assert s.layout["schedule"] == gpu.Session.SCHEDULES[mode]
            assert s.layout["dynamic"] == (1 if mode == "dynamic" else 0)
            it, err, conv = s.iterate(k, KNEVER)
            assert it == k
            out[name] = (s.plan(), s.factors(), s.col_sums())
        assert_parity(out[name][0], ref.plan, rpd, cpd, f"{m}x{n} {name}")
        np.testing.assert_allclose(out[name][1].alpha, ref.alpha, rtol=1e-10)
    for x, y in (("u1", "u2"), ("w1", "w2")):
        assert np.array_equal(out[x][0], out[y][0])
        np.testing.assert_array_equal(out[x][1].alpha, out[y][1].alpha)
        np.testing.assert_array_equal(out[x][2], out[y][2])


@pytest.mark.parametrize("m,n,dt", [(4099, 8192, np.float32), (3001, 8200, np.float32), (2100, 4100, np.float64)])
def test_alternating_sweeps_keep_rows_in_l2(gpu, orc, m, n, dt):
    """Streaming problems (> 64 MiB) store each CTA's last batches L2-resident and
    walk the static row blocks in alternating directions (SweepArgs::keep): the
    direction follows the iteration count, so k iterations in one call, in
    single-iteration calls, or across a resume give the same bits, and every
    count meets the parity bar (odd and even: the backward sweep is the last)."""
    a, rpd, cpd = orc.gen_problem(21, m, n, dtype=dt)
    for k in (3, 4):
        ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 4)
        plans = []
        for chunks in ([k], [1] * k, [2, k - 2]):
            p, f, cs, done, err, conv, lay = run(gpu, a, rpd, cpd, 1.0, 0.1, k, chunks=chunks)
            assert done == k and lay["keep_batches"] > 0 and lay["evict_first"] == 1
            plans.append((p, f.alpha, f.beta, cs))
        assert_parity(plans[0][0], ref.plan, rpd, cpd, f"{m}x{n} {np.dtype(dt).name} K={k}")
        np.testing.assert_allclose(plans[0][1], ref.alpha, rtol=1e-10)
        for other in plans[1:]:
            for x, y in zip(plans[0], other):
                assert np.array_equal(x, y)


@pytest.mark.parametrize("m,n", [(600, 8192), (200, 32768), (900, 4096), (500, 20000)])
def test_split_roles_exact_path(gpu, orc, m, n):
    """The split sweep roles (V >= 2 slices: 8192 columns G = 1, 32768 G = 4, 4096
    columns in 2-row batches, 20000 partial slices G = 3) on inputs that fail the
    fast-path screen — subnormal, zero-adjacent and huge entries — and on rows whose
    factor leaves the certified range: the sweep-1 warps' exact-path masks reach
    their sweep-2 partners and the plan stays bit-identical to the oracle."""
    a, rpd, cpd = orc.gen_problem(91, m, n)
    a[3, 5] = np.float32(1e-40)                     # subnormal input
    a[7, n - 1] = np.float32(2e-38)                 # product underflows after scaling
    a[m // 2, n // 3] = np.float32(3e37)            # product overflows the screen window
    a[m - 2, :] *= np.float32(1e-30)                # a row whose factor leaves [2^-20, 2^20]
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 4, 4)
    p, f, cs, done, err, conv, lay = run(gpu, a, rpd, cpd, 1.0, 0.1, 4, resident=False)
    assert lay["resident"] == 0 and done == 4
    assert np.array_equal(p, ref.plan), f"{m}x{n}: max rel {np.max(np.abs(p.astype(np.float64) - ref.plan) / ref.plan):.3e}"
    np.testing.assert_allclose(f.alpha, ref.alpha, rtol=1e-12)


@pytest.mark.slow
def test_default_schedule_is_bit_reproducible_at_scale(gpu):
    """Two default runs (separate sessions) of problems far past the 64 MiB
    threshold give identical bits: plan, factors, carried column sums and error
    (the reference's promise, fused.hpp:193-196, 242-248); G = 3, 4 and 1."""
    for (m, n, k) in [(16384, 20000, 6), (8192, 32768, 5), (65536, 4096, 5)]:
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
            assert np.array_equal(np.asarray(x), np.asarray(y)), f"{m}x{n}"


def test_calibration_leaves_the_session_state(gpu, orc):
    """uot_calibrate_schedule runs on a scratch copy: plan, factors, column sums
    and the iteration count are unchanged, and the weighted solve continues
    exactly where the session was (== the uniform solve to the parity bar)."""
    m, n = 20000, 4096
    a, rpd, cpd = orc.gen_problem(3, m, n)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 5, 4)
    with gpu.Session(m, n) as s:
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.1))
        s.init_col_sums()
        s.iterate(2, KNEVER)
        before = (s.plan(), s.factors(), s.col_sums(), s.report())
        w = s.calibrate_schedule(4)
        after = (s.plan(), s.factors(), s.col_sums(), s.report())
        assert w.size == s.layout["groups"] and w.min() >= 1 and s.layout["pinned"] == 1
        assert np.array_equal(before[0], after[0]) and np.array_equal(before[2], after[2])
        np.testing.assert_array_equal(before[1].alpha, after[1].alpha)
        np.testing.assert_array_equal(before[1].beta, after[1].beta)
        assert before[3] == after[3]
        it, err, conv = s.iterate(3, KNEVER)
        assert it == 3
        smid, nb, gw = s.schedule_stats()
        assert len(set(smid.tolist())) == smid.size and np.array_equal(gw, w)
        assert_parity(s.plan(), ref.plan, rpd, cpd, "weighted after calibration")
