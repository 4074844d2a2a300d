"""Parity of the sm_100a path (through the C ABI) with the reference CPU solver.

Bar (BASELINE.json north_star): max relative error <= 1e-5 on P and on both
marginal errors after K iterations, on identical synthetic inputs. The sweep
reproduces the reference arithmetic exactly (f64 products rounded once to fp32,
f64 sums of stored values), so the plan is expected to be bit-identical; the
tests enforce the 1e-5 bar and report the bitwise match.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

from conftest import KNEVER, er_ep

pytestmark = pytest.mark.gpu
TOL = 1e-5


def marginal_errors(plan, rpd, cpd):
    p = plan.astype(np.float64)
    return np.max(np.abs(p.sum(axis=1) - rpd)), np.max(np.abs(p.sum(axis=0) - cpd))


def assert_parity(plan, ref_plan, rpd, cpd, what=""):
    rel = np.max(np.abs(plan.astype(np.float64) - ref_plan) / np.abs(ref_plan))
    assert rel <= TOL, f"{what}: max rel err on P {rel:.3e}"
    er_g, ec_g = marginal_errors(plan, rpd, cpd)
    er_r, ec_r = marginal_errors(ref_plan, rpd, cpd)
    # relative 1e-5 on the marginal errors, with an absolute floor at the f64
    # rounding level of the marginals (a converged fp64 plan's errors ARE noise)
    floor = 1e-13 * max(float(np.max(rpd)), float(np.max(cpd)))
    assert abs(er_g - er_r) <= TOL * er_r + floor, f"{what}: row marginal error {er_g} vs {er_r}"
    assert abs(ec_g - ec_r) <= TOL * ec_r + floor, f"{what}: col marginal error {ec_g} vs {ec_r}"
    return rel


def solve(uot, a, rpd, cpd, er, ep, k, tol=KNEVER):
    with uot.Session(a.shape[0], a.shape[1]) as s:
        s.set_problem(uot.Problem(a, rpd, cpd, er, ep))
        s.init_col_sums()
        it, err, conv = s.iterate(k, tol)
        return s.plan(), s.factors(), s.col_sums(), it, err, conv, s.layout


# ------------------------------------------------------- golden (reference) --

def test_golden_small_cases(gpu, orc, small_golden):
    data, meta = small_golden
    bitwise = 0
    for case in meta:
        key = case["key"]
        if case.get("kat"):
            a, rpd, cpd = data[key + "_a"], data[key + "_rpd"], data[key + "_cpd"]
        else:
            a, rpd, cpd = orc.gen_problem(case["seed"], case["rows"], case["cols"])
        plan, f, cs, it, err, conv, lay = solve(gpu, a, rpd, cpd, case["er"], case["ep"], case["iterations"])
        assert it == case["iterations"], key
        if key + "_plan" in data:
            ref_plan = data[key + "_plan"]
            assert_parity(plan, ref_plan, rpd, cpd, key)
            bitwise += int(np.array_equal(plan, ref_plan))
        else:
            rows = data[key + "_rows"]
            rel = np.max(np.abs(plan[rows].astype(np.float64) - data[key + "_plan_rows"]) / data[key + "_plan_rows"])
            assert rel <= TOL, key
            assert abs(plan.astype(np.float64).sum() - data[key + "_plan_sum"][0]) <= 1e-9 * data[key + "_plan_sum"][0]
            bitwise += int(hashlib.sha256(plan.tobytes()).digest() == bytes(data[key + "_plan_sha256"]))
        np.testing.assert_allclose(f.alpha, data[key + "_alpha"], rtol=1e-12, err_msg=key)
        np.testing.assert_allclose(f.beta, data[key + "_beta"], rtol=1e-12, err_msg=key)
        ref_err = data[key + "_err"][0]
        assert abs(err - ref_err) <= TOL * max(ref_err, 1e-300) or (ref_err == 0 and err == 0), key
        if key + "_colsums" in data:
            np.testing.assert_allclose(cs, data[key + "_colsums"], rtol=1e-12, err_msg=key)
    # every golden case reproduced bit for bit (the arithmetic is the reference's)
    assert bitwise == len(meta)


@pytest.mark.slow
def test_golden_big_anchors(gpu, big_golden):
    """BASELINE.json sizes, problem generated in HBM (bit-identical to gen_problem_t)."""
    data, meta = big_golden
    for case in meta:
        key, m, n, k = case["key"], case["rows"], case["cols"], case["iterations"]
        with gpu.Session(m, n) as s:
            s.generate_problem(case["seed"], case["er"], case["ep"])
            s.init_col_sums()
            it, err, conv = s.iterate(k, KNEVER)
            assert it == k
            f = s.factors()
            cs = s.col_sums()
            plan = s.plan()
        rows = data[key + "_rows"]
        ref_rows = data[key + "_plan_rows"]
        assert np.max(np.abs(plan[rows].astype(np.float64) - ref_rows) / ref_rows) <= TOL, key
        # factors and column sums: f64 sums over ~10^4-10^5 terms whose order
        # follows the dynamic batch schedule (which CTA took which rows), so
        # they agree to a few 1e-12 rather than bit for bit
        st = int(data[key + "_alpha_stride"][0])
        np.testing.assert_allclose(f.alpha[::st], data[key + "_alpha_strided"], rtol=1e-10, err_msg=key)
        cst = int(data[key + "_col_stride"][0])
        np.testing.assert_allclose(f.beta[::cst], data[key + "_beta_strided"], rtol=1e-10, err_msg=key)
        np.testing.assert_allclose(cs[::cst], data[key + "_colsums_strided"], rtol=1e-10, err_msg=key)
        total = plan.astype(np.float64).sum()
        assert abs(total - data[key + "_sum"][0]) <= 1e-9 * data[key + "_sum"][0], key
        assert abs(err - data[key + "_err"][0]) <= TOL * data[key + "_err"][0], key
        assert f.alpha[0] == pytest.approx(case["alpha0"], rel=1e-14)
        same = hashlib.sha256(plan.tobytes()).hexdigest() == case["sha256_plan"]
        print(f"{key}: plan bit-identical to the reference: {same}")


# ------------------------------------------------------------ shapes / edges --

@pytest.mark.parametrize("m,n,fi,k", [
    (1, 1, 0.5, 5), (1, 5000, 1 / 1.1, 6), (5000, 1, 1 / 1.1, 6), (3, 7, 1.0, 9),
    (1000, 5000, 0.8, 12),     # G == 1, slice not a multiple of the thread tile
    (200, 8193, 1 / 1.1, 8),   # just past one CTA per row: G = 2, ragged
    (150, 20000, 1 / 1.1, 8),  # G = 3
    (64, 32768, 1 / 1.1, 8),   # G = 4, the headline row width
    (147, 1024, 0.5, 20),      # fewer rows than SMs
    (4099, 4096, 1 / 1.1, 10), # tall, B = 2 rows per batch, odd row count
])
def test_shapes_against_oracle(gpu, orc, m, n, fi, k):
    a, rpd, cpd = orc.gen_problem(1000 + m, m, n)
    er, ep = er_ep(fi)
    plan, f, cs, it, err, conv, lay = solve(gpu, a, rpd, cpd, er, ep, k)
    ref = orc.fused_solve(a, rpd, cpd, er, ep, KNEVER, k, workers=4)
    assert it == k
    assert_parity(plan, ref.plan, rpd, cpd, f"{m}x{n} G={lay['G']}")
    assert abs(err - ref.final_error) <= TOL * ref.final_error
    np.testing.assert_allclose(f.alpha, ref.alpha, rtol=1e-12)
    np.testing.assert_allclose(f.beta, ref.beta, rtol=1e-12)


def test_device_generator_is_bit_exact(gpu, orc):
    for (m, n) in [(33, 70), (300, 20000), (1024, 1024)]:
        a, rpd, cpd = orc.gen_problem(42, m, n)
        with gpu.Session(m, n) as s:
            s.generate_problem(42, 1.0, 1.0)
            assert np.array_equal(s.plan(), a)


def test_seed_col_sums(gpu, orc):
    a, rpd, cpd = orc.gen_problem(3, 777, 9000)
    with gpu.Session(777, 9000) as s:
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 1.0))
        s.init_col_sums()
        np.testing.assert_allclose(s.col_sums(), orc.init_col_sums(a), rtol=1e-14)


# ------------------------------------------------------- KATs and semantics --

def test_hand_checked_iteration(gpu):
    # test_fused.cpp:38-56: beta=[1.5,1.5], alpha=[4/3,2/3], P=[[2,2],[1,1]], col sums [3,3], error 0.5
    a = np.ones((2, 2), np.float32)
    with gpu.Session(2, 2) as s:
        s.set_problem(gpu.Problem(a, np.array([4.0, 2.0]), np.array([3.0, 3.0]), 1.0, 0.0))
        s.init_col_sums()
        np.testing.assert_array_equal(s.col_sums(), [2.0, 2.0])
        it, err, conv = s.iterate(1, KNEVER)
        f = s.factors()
        np.testing.assert_array_equal(f.beta, [1.5, 1.5])
        np.testing.assert_allclose(f.alpha, [4 / 3, 2 / 3], rtol=1e-15)
        np.testing.assert_array_equal(s.plan(), [[2, 2], [1, 1]])
        np.testing.assert_allclose(s.col_sums(), [3.0, 3.0], rtol=1e-14)
        assert err == pytest.approx(0.5, rel=1e-15)


def test_fixed_point(gpu):
    # test_fused.cpp:58-66 and :210-220
    a = np.ones((6, 9), np.float32)
    r = gpu.fused_solve(gpu.Problem(a, np.full(6, 9.0), np.full(9, 6.0), 1.0, 1.0), 1e-9, 50)
    assert r.report.converged and r.report.iterations == 1 and r.report.final_error == 0.0
    np.testing.assert_array_equal(r.plan, a)


def test_convergence_stops_at_the_reference_iteration(gpu, orc):
    # test_fused.cpp:222-231, acceptance c08: balanced masses, same stopping iteration
    for seed, m, n in [(37, 24, 24), (5, 300, 9000)]:
        a, rpd, cpd = orc.gen_problem(seed, m, n)
        cpd = cpd * (rpd.sum() / cpd.sum())
        ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.0, 1e-6, 10000, 1)
        r = gpu.fused_solve(gpu.Problem(a, rpd, cpd, 1.0, 0.0), 1e-6, 10000)
        assert ref.converged and r.report.converged
        assert r.report.iterations == ref.iterations
        assert_parity(r.plan, ref.plan, rpd, cpd, "converged")


def test_iterate_is_resumable(gpu, orc):
    # k iterations in one call == several calls (device-resident state carries over)
    a, rpd, cpd = orc.gen_problem(8, 500, 3000)
    with gpu.Session(500, 3000) as s:
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.1))
        s.init_col_sums()
        for _ in range(3):
            s.iterate(4, KNEVER)
        p1 = s.plan()
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.1))  # reset, run 12 at once
        s.init_col_sums()
        s.iterate(12, KNEVER)
        assert np.array_equal(p1, s.plan())
        assert s.report()[0] == 12


def test_deterministic(gpu, orc):
    a, rpd, cpd = orc.gen_problem(9, 256, 40000)
    p1 = solve(gpu, a, rpd, cpd, 1.0, 0.1, 7)[0]
    p2 = solve(gpu, a, rpd, cpd, 1.0, 0.1, 7)[0]
    assert np.array_equal(p1, p2)


def test_fused_iterate_host_api(gpu, orc):
    # fused_iterate (fused.hpp:164-191): host matrix + FusedState updated in place, fi passed directly
    a, rpd, cpd = orc.gen_problem(31, 64, 96)
    fi = 0.5
    p = gpu.Problem(a, rpd, cpd, 1.0, 1.0)
    mine = a.copy()
    st = gpu.FusedState(orc.init_col_sums(mine))
    theirs = a.copy()
    cs = orc.init_col_sums(theirs)
    for _ in range(5):
        f = gpu.fused_iterate(mine, st, p, fi)
        alpha, beta = orc.fused_iterate(theirs, cs, rpd, cpd, fi)
        np.testing.assert_allclose(f.alpha, alpha, rtol=1e-13)
        np.testing.assert_allclose(f.beta, beta, rtol=1e-13)
    assert_parity(mine, theirs, rpd, cpd, "fused_iterate")
    np.testing.assert_allclose(st.col_sums, cs, rtol=1e-13)


def test_degenerate_sums_raise(gpu, orc):
    # test_fused.cpp:233-241: zero carried column sums -> DegenerateSum, plan untouched
    a, rpd, cpd = orc.gen_problem(38, 4, 4)
    with gpu.Session(4, 4) as s:
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 1.0))
        s.set_col_sums(np.zeros(4))
        with pytest.raises(gpu.DegenerateSum):
            s.iterate(1, KNEVER)
        np.testing.assert_array_equal(s.plan(), a)
        with pytest.raises(gpu.InvalidParameter):
            s.set_col_sums(np.ones(3))


def test_invalid_problems_rejected(gpu, orc):
    a, rpd, cpd = orc.gen_problem(25, 6, 6)
    bad = a.copy()
    bad[2, 3] = -1.0
    for aa, rr in [(bad, rpd), (a, np.where(np.arange(6) == 3, 0.0, rpd))]:
        with pytest.raises(gpu.InvalidParameter):
            gpu.fused_solve(gpu.Problem(aa, rr, cpd, 1.0, 1.0), 1e-6, 10)
    with pytest.raises(gpu.InvalidParameter):
        gpu.fused_solve(gpu.Problem(a, rpd, cpd, 0.0, 1.0), 1e-6, 10)


def test_subnormal_entries_exact(gpu, orc):
    # the fast f32->f64 path is screened; zero/subnormal inputs take the exact route
    a, rpd, cpd = orc.gen_problem(77, 64, 2048)
    a[3, 5] = np.float32(1e-40)   # subnormal input
    a[7, 9] = np.float32(2e-38)   # product underflows to subnormal after scaling
    plan, f, cs, it, err, conv, lay = solve(gpu, a, rpd, cpd, 1.0, 0.1, 6)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 6, 1)
    assert np.array_equal(plan, ref.plan)


def test_single_rank_distributed_session(gpu, orc):
    # distributed_solve with one rank (test_distributed.cpp:92-104): no NCCL, CommStats kept
    from paper_2412_11079_b200 import distributed as D
    a, rpd, cpd = orc.gen_problem(11, 32, 32)
    r = D.distributed_solve(gpu.Problem(a, rpd, cpd, 1.0, 1.0), KNEVER, 25)
    ref = orc.distributed_solve(a, rpd, cpd, 1.0, 1.0, KNEVER, 25, 1)
    assert r.report.iterations == 25 and r.report.solver == "dist"
    assert r.comm.allreduce_calls == 25 and r.comm.doubles_reduced == 25 * 32
    assert_parity(r.plan, ref.plan, rpd, cpd, "dist1")


# ----------------------------------------------- size-independent properties --

@pytest.mark.slow
def test_full_size_properties(gpu):
    """131072 x 32768 (16 GiB, BASELINE config 5 on one GPU): with fi = 1 the row
    pass makes every row sum equal its marginal; the carried column sums equal
    the column sums of the resident plan; a rerun is bit-identical."""
    m, n = 131072, 32768
    rows = np.sort(np.random.default_rng(0).choice(m, 48, replace=False))
    rpd = np.array([gpu.gen_block(42, m, n, int(i), 1).rpd[0] for i in rows])
    with gpu.Session(m, n) as s:
        s.generate_problem(42, 1.0, 0.0)  # fi = 1: plain normalisation
        s.init_col_sums()
        s.iterate(3, KNEVER)
        plan = s.plan()
        cs = s.col_sums()
        f = s.factors()
        rs = plan[rows].sum(axis=1, dtype=np.float64)
        np.testing.assert_allclose(rs, rpd, rtol=1e-6)  # each stored entry carries one fp32 rounding
        np.testing.assert_allclose(cs, plan.sum(axis=0, dtype=np.float64), rtol=1e-9)
        assert np.all(np.isfinite(f.alpha)) and np.all(f.alpha > 0)
        s.generate_problem(42, 1.0, 0.0)
        s.init_col_sums()
        s.iterate(3, KNEVER)
        assert np.array_equal(plan[rows], s.plan()[rows])


@pytest.mark.parametrize("m,n,k", [(40, 300000, 4), (9, 600000, 3)])
def test_very_wide_rows(gpu, orc, m, n, k):
    # G = ceil(cols / 8192) > 32 CTAs share a row: the exchange gathers the
    # group's records 32 lanes at a time (no column limit below #SMs x 8192)
    a, rpd, cpd = orc.gen_problem(17, m, n)
    plan, f, cs, it, err, conv, lay = solve(gpu, a, rpd, cpd, 1.0, 0.1, k)
    assert lay["G"] > 32 and it == k
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 4)
    assert_parity(plan, ref.plan, rpd, cpd, f"{m}x{n}")
    np.testing.assert_allclose(f.alpha, ref.alpha, rtol=1e-12)


def test_randomized_shapes_against_oracle(gpu, orc):
    # seeded sweep over shapes, damping and iteration counts that exercise every
    # layout: G = 1 with 1..8 rows per batch, G > 1, ragged slices, resident and
    # streaming modes, fi < 1 and fi = 1
    rng = np.random.default_rng(2024)
    for case in range(24):
        m = int(rng.integers(1, 700))
        n = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(300, 9000)), int(rng.integers(9000, 40000))]))
        fi = float(rng.choice([1.0, 0.5, 1 / 1.1, 0.9]))
        k = int(rng.integers(1, 12))
        er, ep = er_ep(fi)
        a, rpd, cpd = orc.gen_problem(int(rng.integers(0, 2**31)), m, n)
        plan, f, cs, it, err, conv, lay = solve(gpu, a, rpd, cpd, er, ep, k)
        ref = orc.fused_solve(a, rpd, cpd, er, ep, KNEVER, k, 3)
        assert it == k, (case, m, n)
        assert_parity(plan, ref.plan, rpd, cpd, f"case {case}: {m}x{n} fi={fi} k={k} layout={lay}")
        assert abs(err - ref.final_error) <= 1e-9 * max(1.0, ref.final_error), (case, m, n)


@pytest.mark.parametrize("m,n,dt", [(3, 148 * 8192 + 100, np.float32), (2, 148 * 4096 + 7, np.float64)])
def test_rows_wider_than_the_grid_run_two_pass(gpu, orc, m, n, dt):
    # G > #SMs: one row cannot span the sweep grid; the session runs the paper's
    # two-pass schedule (tiled.hpp:210-229) for the seed and every iteration
    uot = gpu
    a, rpd, cpd = orc.gen_problem(21, m, n, dtype=dt)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 3, 1)
    with uot.Session(m, n, dtype=dt) as s:
        assert s.layout["variant"] == 1  # UOT_VARIANT_TWO_PASS
        s.set_problem(uot.Problem(a, rpd, cpd, 1.0, 0.1))
        s.init_col_sums()
        np.testing.assert_allclose(s.col_sums(), a.astype(np.float64).sum(0), rtol=1e-12)
        it, err, _ = s.iterate(3, KNEVER)
        plan = s.plan()
        with pytest.raises(uot.ConfigError):
            s.set_variant("fused")
    assert it == 3
    rel = np.max(np.abs(plan.astype(np.float64) - ref.plan) / ref.plan)
    assert rel <= (1e-12 if dt == np.float64 else 1e-5), rel
    assert abs(err - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)


def test_baseline_config2_full_size_bitwise_vs_reference(gpu, ref):
    # BASELINE config 2 at its full size and iteration count (8192^2, K=500) against the
    # reference's own fused_solve (oracle/_ref, all host threads): identical plans
    # (tools/full_parity.py runs configs 3 and 4 too: profiles/r01_full_parity.json)
    import oracle
    uot = gpu
    a, rpd, cpd = oracle.Oracle().gen_problem(42, 8192, 8192, threads=os.cpu_count() or 1)
    r = ref.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 500, os.cpu_count() or 1)
    g = uot.fused_solve(uot.Problem(a, rpd, cpd, 1.0, 0.1), KNEVER, 500)
    assert g.report.iterations == r.iterations == 500
    assert np.array_equal(g.plan, r.plan)
    np.testing.assert_allclose(g.factors.beta, r.beta, rtol=1e-12)


def test_concurrent_sessions_in_threads(gpu, orc):
    # independent sessions on one GPU from several host threads (ctypes drops the GIL):
    # their sweeps interleave on the device; G > 1 launches stay cooperative so the
    # SM-id-addressed CTAs of each grid remain a permutation (the seed included)
    import threading
    uot = gpu
    cases = [(40, 32768, 5, 1), (64, 16384, 6, 2), (300, 3000, 7, 3), (5000, 1000, 4, 4)]
    out, errs = {}, []

    def work(m, n, k, seed):
        try:
            a, rpd, cpd = orc.gen_problem(seed, m, n)
            out[seed] = (uot.fused_solve(uot.Problem(a, rpd, cpd, 1.0, 0.1), KNEVER, k),
                         orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 2))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    for _ in range(2):
        ts = [threading.Thread(target=work, args=c) for c in cases]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errs, errs
        for seed, (g, r) in out.items():
            rel = np.max(np.abs(g.plan.astype(np.float64) - r.plan) / r.plan)
            assert rel <= 1e-5 and g.report.iterations == r.iterations, (seed, rel)


def test_set_col_sums_after_convergence(gpu, orc):
    """A converged session given a new FusedState (uot_set_col_sums) runs again:
    beta is recomputed from the caller's sums and the next iteration equals the
    reference's fused_iterate from that state (fused.hpp:164-191)."""
    a, rpd, cpd = orc.gen_problem(37, 48, 64)
    cpd = cpd * (rpd.sum() / cpd.sum())
    with gpu.Session(48, 64) as s:
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.0))
        s.init_col_sums()
        it, err, conv = s.iterate(10000, 1e-6)
        assert conv
        plan = s.plan()
        cs = orc.init_col_sums(plan)  # a different (exact seed) state than the carried one
        s.set_col_sums(cs)
        it2, err2, conv2 = s.iterate(1, 1e-300)
        assert it2 == 1
        got = s.plan()
        f = s.factors()
    ref_plan = plan.copy()
    ref_cs = cs.copy()
    fi = orc.compute_fi(1.0, 0.0)
    _, rbeta = orc.fused_iterate(ref_plan, ref_cs, rpd, cpd, fi, 1)
    np.testing.assert_allclose(f.beta, rbeta, rtol=1e-14)
    assert_parity(got, ref_plan, rpd, cpd, "after set_col_sums")
