"""The reference's in-process distributed_solve (distributed.hpp:52-142) on the GPU:
uot.distributed_solve(p, tol, max_iter, ranks | RankPartition) drives every rank
from ONE process (uot_create_group / uot_group_*), here with all ranks sharing
cuda:0. Checked against the oracle's distributed_solve, which is bitwise
fused_solve with P workers (test_distributed.cpp:106-118).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import KNEVER

pytestmark = pytest.mark.gpu


def _problem(uot, orc, seed, rows, cols, balance=False, ep=0.1):
    a, rpd, cpd = orc.gen_problem(seed, rows, cols)
    if balance:
        cpd = cpd * (rpd.sum() / cpd.sum())
    return a, rpd, cpd, uot.Problem(a, rpd, cpd, 1.0, ep)


def _assert_matches(res, ref, k):
    assert res.report.iterations == ref.iterations == k
    rel = np.max(np.abs(res.plan.astype(np.float64) - ref.plan) / ref.plan)
    assert rel <= 1e-5, f"max rel err {rel:.3e}"
    np.testing.assert_allclose(res.factors.alpha, ref.alpha, rtol=1e-12)
    np.testing.assert_allclose(res.factors.beta, ref.beta, rtol=1e-12)
    assert abs(res.report.final_error - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)


@pytest.mark.parametrize("ranks,rows,cols,k", [(2, 300, 2000, 10), (3, 257, 1000, 8), (2, 64, 20000, 6),
                                               (4, 96, 8192, 5), (2, 64, 32768, 4), (2, 100, 16384, 4)])
def test_group_matches_distributed_solve(gpu, orc, ranks, rows, cols, k):
    uot = gpu
    a, rpd, cpd, p = _problem(uot, orc, 42, rows, cols)
    ref = orc.distributed_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, ranks)
    res = uot.distributed_solve(p, KNEVER, k, ranks, devices=[0] * ranks)
    _assert_matches(res, ref, k)
    assert res.comm.allreduce_calls == k and res.comm.doubles_reduced == k * cols
    assert res.report.solver == "dist"


def test_group_stops_at_the_reference_iteration(gpu, orc):
    uot = gpu
    a, rpd, cpd, p = _problem(uot, orc, 5, 300, 9000, balance=True, ep=0.0)
    ref = orc.distributed_solve(a, rpd, cpd, 1.0, 0.0, 1e-6, 10000, 2)
    res = uot.distributed_solve(p, 1e-6, 10000, 2, devices=[0, 0])
    assert ref.converged and res.report.converged
    assert res.report.iterations == ref.iterations


def test_group_custom_partition(gpu, orc):
    uot = gpu
    a, rpd, cpd, p = _problem(uot, orc, 9, 300, 3000)
    part = uot.RankPartition(3, [(0, 10), (10, 200), (200, 300)])  # unbalanced, contiguous, covering
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 7, workers=3)  # same rows, other summation blocks
    res = uot.distributed_solve(p, KNEVER, 7, part, devices=[0, 0, 0])
    rel = np.max(np.abs(res.plan.astype(np.float64) - ref.plan) / ref.plan)
    assert rel <= 1e-5 and res.report.iterations == 7
    np.testing.assert_allclose(res.factors.alpha, ref.alpha, rtol=1e-12)


def test_group_rejects_bad_partitions(gpu, orc):
    uot = gpu
    _, _, _, p = _problem(uot, orc, 1, 40, 300)
    with pytest.raises(uot.PartitionError):
        uot.distributed_solve(p, KNEVER, 2, uot.RankPartition(2, [(0, 10), (10, 30)]))  # does not cover
    with pytest.raises(uot.PartitionError):
        uot.distributed_solve(p, KNEVER, 2, uot.RankPartition(2, [(0, 0), (0, 40)]))  # empty block
    with pytest.raises(uot.PartitionError):
        uot.distributed_solve(p, KNEVER, 2, 41)  # more ranks than rows (plan.cpp:36-39)
    with pytest.raises(uot.InvalidParameter):
        uot.distributed_solve(p, 0.0, 2, 2)


def test_group_ranks_refuse_single_rank_collectives(gpu, orc):
    uot = gpu
    a, rpd, cpd, p = _problem(uot, orc, 2, 50, 700)
    with uot.SessionGroup(50, 700, 2, devices=[0, 0]) as g:
        for s in g.ranks:
            b, e = s.row_offset, s.row_offset + s.rows
            s.set_problem(uot.Problem(a[b:e], rpd[b:e], cpd, 1.0, 0.1))
        with pytest.raises(uot.InvalidParameter):
            g.ranks[0].init_col_sums()  # would wait on rank 1 forever: refused
        g.init_col_sums()
        with pytest.raises(uot.InvalidParameter):
            g.ranks[1].iterate(1)
        it, _, _ = g.iterate(3)
        assert it == 3
        it, _, _ = g.iterate(2)  # resumable, like Session.iterate
        assert it == 2 and g.ranks[0].report()[0] == 5


def test_group_f64_matches_oracle(gpu, orc):
    uot = gpu
    a, rpd, cpd = orc.gen_problem(11, 200, 6000, dtype=np.float64)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 6, 2)
    res = uot.distributed_solve(uot.Problem(a, rpd, cpd, 1.0, 0.1), KNEVER, 6, 2, devices=[0, 0])
    assert res.plan.dtype == np.float64 and res.report.iterations == 6
    rel = np.max(np.abs(res.plan - ref.plan) / ref.plan)
    assert rel <= 1e-12, f"f64 plan differs by {rel:.3e}"
    np.testing.assert_allclose(res.factors.beta, ref.beta, rtol=1e-12)


def test_group_device_list_must_match_ranks(gpu):
    uot = gpu
    with pytest.raises(uot.InvalidParameter):
        uot.SessionGroup(100, 100, 3, devices=[0, 0])


def test_group_rows_wider_than_the_grid_are_refused(gpu, orc):
    # G > #SMs is served by the two-pass schedule on ONE rank; the ablation
    # schedules have no cross-rank exchange, so a multi-rank group refuses it
    uot = gpu
    with pytest.raises(uot.ConfigError):
        uot.SessionGroup(4, 148 * 8192 + 100, 2, devices=[0, 0])


def test_group_collectives_reject_ranks_of_different_groups(gpu):
    uot = gpu
    with uot.SessionGroup(40, 300, 2, devices=[0, 0]) as g1, uot.SessionGroup(40, 300, 2, devices=[0, 0]) as g2:
        import ctypes as C
        # every rank has a problem, so only the group check can refuse the call
        # (without it rank 1 of g2 would wait for a peer of g1 that never publishes)
        for g in (g1, g2):
            for s in g.ranks:
                s.generate_problem(3, 1.0, 0.1)
        mixed = (C.c_void_p * 2)(g1.ranks[0]._h.value, g2.ranks[1]._h.value)
        rc = uot.lib().uot_group_init_col_sums(C.cast(mixed, C.c_void_p), 2)
        assert rc == 1  # UOT_INVALID_PARAMETER, no hang on a peer that never publishes
        assert "session group" in g2.ranks[1]._err()
        it, err, conv = C.c_uint64(), C.c_double(), C.c_int()
        rc = uot.lib().uot_group_iterate(C.cast(mixed, C.c_void_p), 2, 3, 1e-300, C.byref(it), C.byref(err),
                                         C.byref(conv))
        assert rc == 1 and "session group" in g2.ranks[1]._err()
        g1.init_col_sums()  # the groups themselves still work
        assert g1.iterate(2)[0] == 2
