"""The CPU oracle (oracle/uot_oracle.c) pinned against the reference itself
(oracle/_ref) and the golden vectors it produced. Mirrors the reference suites
proj/tests/test_scaling.cpp, test_fused.cpp, test_distributed.cpp, test_io.cpp."""
from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from conftest import KNEVER, er_ep

# ------------------------------------------------------------ generator --


def ref_splitmix64(state):
    """Independent transcription (test_io.cpp:22-29 style) of rng.hpp:14-20."""
    state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    return state, z ^ (z >> 31)


def test_splitmix64_pinned_sequence(orc):
    import ctypes as C
    for seed in (0, 1, 42, 1 << 63):
        st = C.c_uint64(seed)
        ref_state = seed
        for _ in range(20):
            ref_state, want = ref_splitmix64(ref_state)
            assert orc.lib.orc_splitmix64_next(C.byref(st)) & (2**64 - 1) == want


def test_generator_fill_order_and_unit_range(orc):
    # test_io.cpp:64-97: A row-major, then rpd, then cpd, all (0,1]; fp32 = cast of the draw
    a, rpd, cpd = orc.gen_problem(11, 4, 5)
    state = 11
    draws = []
    for _ in range(4 * 5 + 4 + 5):
        state, z = ref_splitmix64(state)
        draws.append(((z >> 11) + 1) * 2.0**-53)
    assert np.array_equal(a.ravel(), np.array(draws[:20], np.float32))
    assert np.array_equal(rpd, np.array(draws[20:24]))
    assert np.array_equal(cpd, np.array(draws[24:]))
    assert (a > 0).all() and (a <= 1).all()


def test_generator_matches_reference(orc, ref):
    for (seed, m, n) in [(42, 1024, 1024), (3, 5, 4), (7, 33, 70)]:
        mine = orc.gen_problem(seed, m, n, threads=4)
        theirs = ref.gen_problem(seed, m, n)
        for x, y in zip(mine, theirs):
            assert np.array_equal(x, y)


# -------------------------------------------------------------- scalars --


def test_compute_fi(orc, ref):
    # test_scaling.cpp:11-27
    for er, ep, want in [(1, 1, 0.5), (3, 1, 0.75), (1, 0, 1.0), (1, 3, 0.25), (0.5, 0.5, 0.5)]:
        assert orc.compute_fi(er, ep) == want == ref.compute_fi(er, ep)
    import oracle
    for er, ep in [(0, 1), (-1, 1), (1, -0.5), (math.nan, 1), (1, math.inf)]:
        with pytest.raises(oracle.OracleError) as e:
            orc.compute_fi(er, ep)
        assert e.value.code == 1


def test_rescale_factor(orc, ref):
    # test_scaling.cpp:42-58
    for t, s, fi, want in [(4, 1, 0.5, 2.0), (2, 8, 1.0, 0.25), (8, 2, 0.5, 2.0), (5, 5, 0.5, 1.0),
                           (1e-9, 1e-9, 1.0, 1.0), (3, 3, 0.123, 1.0)]:
        assert orc.rescale_factor(t, s, fi) == want == ref.rescale_factor(t, s, fi)
    import oracle
    for t, s in [(1, 0), (1, -2), (1, math.nan), (1e300, 1e-300)]:
        with pytest.raises(oracle.OracleError) as e:
            orc.rescale_factor(t, s, 1.0 if t == 1e300 else 0.5)
        assert e.value.code == 2


def test_rescale_factor_matches_reference_randomly(orc, ref):
    rng = np.random.default_rng(5)
    for _ in range(300):
        t, s = np.exp((rng.random(2) - 0.5) * 40)
        fi = rng.random()
        assert orc.rescale_factor(t, s, fi) == ref.rescale_factor(t, s, fi)


def test_convergence_error(orc):
    # test_scaling.cpp:72-78
    assert orc.convergence_error([1.0, 1.0], [1.0, 1.0, 1.0]) == 0.0
    assert orc.convergence_error([1.1, 0.9], [1.0]) == pytest.approx(0.1, rel=1e-15)
    assert orc.convergence_error([1.0], [0.5]) == 0.5
    assert orc.convergence_error([4 / 3, 2 / 3], [1.5, 1.5]) == pytest.approx(0.5, rel=1e-15)


# ----------------------------------------------------------------- plans --


def test_balanced_blocks_and_rank_partition(orc, ref):
    # test_fused.cpp:88-107, test_distributed.cpp:20-46
    assert orc.balanced_blocks(3, 8) == [0, 3, 6, 8]
    assert orc.balanced_blocks(5, 3) == [0, 1, 2, 3, 3, 3]
    assert orc.rank_partition(8, 8) == list(range(9))
    assert orc.rank_partition(1, 5) == [0, 5]
    import oracle
    for r, m in [(0, 8), (9, 8)]:
        with pytest.raises(oracle.OracleError) as e:
            orc.rank_partition(r, m)
        assert e.value.code == 3
    for r, m in [(3, 8), (7, 100), (8, 131072), (37, 32768)]:
        assert orc.rank_partition(r, m) == ref.rank_partition(r, m)


def test_allreduce_ascending_order(orc):
    # test_distributed.cpp:48-60
    import ctypes as C
    parts = [np.array([1.0, 2.0]), np.array([3.0, 4.0]), np.array([5.0, 6.0])]
    arr = (C.c_void_p * 3)(*[p.ctypes.data for p in parts])
    out = np.empty(2)
    orc.lib.orc_allreduce_vectors(arr, 3, 2, out.ctypes.data_as(C.c_void_p))
    assert list(out) == [9.0, 12.0]


# ------------------------------------------------- the path vs reference --


@pytest.mark.parametrize("seed,m,n,fi,k,w", [
    (21, 16, 16, 0.5, 25, 1), (22, 10, 33, 1.0, 25, 1), (24, 27, 6, 0.75, 25, 1),
    (32, 64, 64, 0.5, 50, 4), (33, 128, 128, 0.5, 100, 16), (42, 1024, 1024, 1 / 1.1, 100, 8),
    (5, 1, 1, 0.5, 7, 1), (6, 3, 200, 0.9, 12, 5),
])
def test_fused_solve_bitwise_equals_reference(orc, ref, seed, m, n, fi, k, w):
    a, rpd, cpd = orc.gen_problem(seed, m, n)
    er, ep = er_ep(fi)
    mine = orc.fused_solve(a, rpd, cpd, er, ep, KNEVER, k, w)
    theirs = ref.fused_solve(a, rpd, cpd, er, ep, KNEVER, k, w)
    assert mine.iterations == theirs.iterations == k
    assert np.array_equal(mine.plan, theirs.plan)
    assert np.array_equal(mine.alpha, theirs.alpha)
    assert np.array_equal(mine.beta, theirs.beta)
    assert mine.final_error == theirs.final_error


def test_solve_to_convergence_matches_reference(orc, ref):
    # test_fused.cpp:222-231 / acceptance c08: balanced masses converge; same iteration
    a, rpd, cpd = orc.gen_problem(37, 24, 24)
    cpd = cpd * (rpd.sum() / cpd.sum())
    # fp32 storage bottoms the factor error out near 1e-7, so tol 1e-6 (the reference test is f64)
    mine = orc.fused_solve(a, rpd, cpd, 1.0, 1.0, 1e-6, 10000, 1)
    theirs = ref.fused_solve(a, rpd, cpd, 1.0, 1.0, 1e-6, 10000, 1)
    assert mine.converged and theirs.converged
    assert mine.iterations == theirs.iterations
    assert np.array_equal(mine.plan, theirs.plan)


def test_distributed_bitwise_equals_reference_and_workers(orc, ref):
    # test_distributed.cpp:106-118 (k ranks == k workers, bit for bit), 142-155 (one allreduce/iter)
    a, rpd, cpd = orc.gen_problem(21, 40, 17)
    for k in (1, 2, 3, 5):
        d = orc.distributed_solve(a, rpd, cpd, 1.0, 1.0, KNEVER, 30, k)
        r = ref.distributed_solve(a, rpd, cpd, 1.0, 1.0, KNEVER, 30, k)
        w = orc.fused_solve(a, rpd, cpd, 1.0, 1.0, KNEVER, 30, k)
        assert np.array_equal(d.plan, r.plan) and np.array_equal(d.plan, w.plan)
        assert np.array_equal(d.alpha, r.alpha) and np.array_equal(d.beta, r.beta)
        assert d.allreduce_calls == r.allreduce_calls == 30
        assert d.doubles_reduced == r.doubles_reduced == 30 * 17


def test_degenerate_and_invalid_inputs(orc):
    import oracle
    a, rpd, cpd = orc.gen_problem(38, 4, 4)
    cs = np.zeros(4)
    with pytest.raises(oracle.OracleError) as e:  # test_fused.cpp:233-241
        orc.fused_iterate(a.copy(), cs, rpd, cpd, 0.5)
    assert e.value.code == 2
    bad = a.copy()
    bad[0, 0] = -1.0
    with pytest.raises(oracle.OracleError) as e:  # test_baseline.cpp:104-113
        orc.fused_solve(bad, rpd, cpd, 1.0, 1.0, 1e-6, 10)
    assert e.value.code == 1
    with pytest.raises(oracle.OracleError):
        orc.fused_solve(a, rpd, cpd, 1.0, 1.0, 0.0, 10)
    with pytest.raises(oracle.OracleError):
        orc.fused_solve(a, rpd, cpd, 1.0, 1.0, 1e-6, 0)


def test_fixed_point_is_bit_identical(orc):
    # test_fused.cpp:58-66
    a = np.ones((6, 9), np.float32)
    r = orc.fused_solve(a, np.full(6, 9.0), np.full(9, 6.0), 1.0, 1.0, 1e-9, 50)
    assert r.converged and r.iterations == 1 and r.final_error == 0.0
    assert np.array_equal(r.plan, a)


def test_unequal_mass_plateau(orc):
    # test_baseline.cpp:142-167: error flattens at max(c, 1/c) - 1
    fi = 0.5
    a, rpd, cpd = orc.gen_problem(10, 12, 12)
    er, ep = er_ep(fi)
    r = orc.fused_solve(a, rpd, cpd, er, ep, KNEVER, 300)
    c = (rpd.sum() / cpd.sum()) ** (fi / (2 - fi))
    assert abs(r.final_error - (max(c, 1 / c) - 1)) < 1e-4


# -------------------------------------------------- golden (reference) --


def test_oracle_matches_golden_small(orc, small_golden):
    data, meta = small_golden
    for case in meta:
        key = case["key"]
        if case.get("kat"):
            r = orc.fused_solve(data[key + "_a"], data[key + "_rpd"], data[key + "_cpd"], case["er"],
                                case["ep"], KNEVER, case["iterations"], 1)
        else:
            a, rpd, cpd = orc.gen_problem(case["seed"], case["rows"], case["cols"])
            r = orc.fused_solve(a, rpd, cpd, case["er"], case["ep"], KNEVER, case["iterations"],
                                case["workers"])
            assert np.array_equal(r.col_sums, data[key + "_colsums"]), key
        if key + "_plan" in data:
            assert np.array_equal(r.plan, data[key + "_plan"]), key
        else:
            assert np.array_equal(r.plan[data[key + "_rows"]], data[key + "_plan_rows"]), key
            assert hashlib.sha256(r.plan.tobytes()).digest() == bytes(data[key + "_plan_sha256"]), key
        assert np.array_equal(r.alpha, data[key + "_alpha"]), key
        assert np.array_equal(r.beta, data[key + "_beta"]), key
        assert r.final_error == data[key + "_err"][0], key


def test_kat_values(small_golden):
    # test_fused.cpp:38-56 hand-checked: beta=[1.5,1.5], alpha=[4/3,2/3], P=[[2,2],[1,1]], error 0.5
    data, _ = small_golden
    assert list(data["kat_2x2_beta"]) == [1.5, 1.5]
    assert data["kat_2x2_alpha"] == pytest.approx([4 / 3, 2 / 3], rel=1e-15)
    assert np.array_equal(data["kat_2x2_plan"], np.array([[2, 2], [1, 1]], np.float32))
    assert data["kat_2x2_err"][0] == pytest.approx(0.5, rel=1e-15)
    assert data["kat_1x1_plan"][0, 0] == 4.0  # test_baseline.cpp:64-74
    assert data["kat_damped_alpha"][0] == 2.0  # (8/2)^0.5, test_baseline.cpp:22-28


def test_survey_anchor_1024(small_golden):
    # 1024^2, K=100, seed 42, fi=1/1.1 (measured on the reference)
    data, _ = small_golden
    key = "s42_1024x1024_k100_w8"
    assert data[key + "_alpha"][0] == 1.011444589094509
    assert data[key + "_beta"][0] == 0.98868490846191781
    assert data[key + "_err"][0] == 0.011444589182068698
