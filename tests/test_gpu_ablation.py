"""The ablation schedules compute the same iteration as the fused sweep.

TWO_PASS (tiled.hpp:210-229, part4 -> alpha -> part2) and BASELINE
(baseline.hpp:100-110, four sweeps) run on the GPU through uot_set_variant and
are checked against the oracle: the two-pass schedule against fused_solve (the
reference's tiled_iterate "carries column sums exactly like the fused solver",
tiled.hpp:206-208) and the baseline against the reference's own baseline_solve
(oracle/_ref) or, without it, against fused_solve (baseline == fused up to
summation order). Bar: 1e-5 relative on P, same stopping iteration.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import KNEVER
from test_gpu_parity import assert_parity

pytestmark = pytest.mark.gpu


def run_variant(uot, variant, a, rpd, cpd, er, ep, k, tol=KNEVER):
    with uot.Session(a.shape[0], a.shape[1]) as s:
        s.set_problem(uot.Problem(a, rpd, cpd, er, ep))
        s.init_col_sums()
        s.set_variant(variant)
        it, err, conv = s.iterate(k, tol)
        return s.plan(), s.factors(), it, err, conv


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 30), (300, 20000, 8), (2000, 513, 20), (4096, 4096, 6), (7, 3, 11)])
@pytest.mark.parametrize("variant", ["two_pass", "baseline"])
def test_variant_matches_oracle(gpu, orc, variant, m, n, k):
    a, rpd, cpd = orc.gen_problem(42, m, n)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 1)
    plan, f, it, err, conv = run_variant(gpu, variant, a, rpd, cpd, 1.0, 0.1, k)
    assert it == k
    assert_parity(plan, ref.plan, rpd, cpd, f"{variant} {m}x{n}")
    np.testing.assert_allclose(f.alpha, ref.alpha, rtol=1e-11)
    np.testing.assert_allclose(f.beta, ref.beta, rtol=1e-11)
    assert abs(err - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)


def test_baseline_matches_reference_baseline_solve(gpu, orc, ref):
    a, rpd, cpd = orc.gen_problem(9, 512, 640)
    r = ref.baseline_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 15)
    plan, f, it, err, conv = run_variant(gpu, "baseline", a, rpd, cpd, 1.0, 0.1, 15)
    assert it == r.iterations == 15
    assert_parity(plan, r.plan, rpd, cpd, "baseline vs reference baseline_solve")
    assert abs(err - r.final_error) <= 1e-9 * max(1.0, r.final_error)


@pytest.mark.parametrize("variant", ["two_pass", "baseline"])
def test_variant_converges_at_the_reference_iteration(gpu, orc, variant):
    a, rpd, cpd = orc.gen_problem(37, 24, 24)
    cpd = cpd * (rpd.sum() / cpd.sum())
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.0, 1e-6, 10000, 1)
    plan, f, it, err, conv = run_variant(gpu, variant, a, rpd, cpd, 1.0, 0.0, 10000, tol=1e-6)
    assert conv and it == ref.iterations
    assert_parity(plan, ref.plan, rpd, cpd, f"{variant} converged")


def test_unknown_variant_rejected(gpu):
    with gpu.Session(8, 8) as s:
        with pytest.raises(gpu.InvalidParameter):
            s.set_variant("three_pass")


@pytest.mark.parametrize("m,n,k", [(300, 2000, 8), (257, 4098, 5), (7, 3, 11), (64, 9001, 4)])
@pytest.mark.parametrize("variant", ["two_pass", "baseline"])
def test_variant_f64_matches_oracle(gpu, orc, variant, m, n, k):
    # Problem<double>: plain f64 products in every schedule (baseline.hpp / tiled.hpp with T = double);
    # 4098 / 9001 columns leave a row pitch that is not a multiple of 4 (per-element bounds)
    a, rpd, cpd = orc.gen_problem(43, m, n, dtype=np.float64)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 2)
    with gpu.Session(m, n, dtype=np.float64) as s:
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.1))
        s.init_col_sums()
        s.set_variant(variant)
        it, err, conv = s.iterate(k, KNEVER)
        plan, f = s.plan(), s.factors()
    assert it == k and plan.dtype == np.float64
    rel = np.max(np.abs(plan - ref.plan) / ref.plan)
    assert rel <= 1e-12, f"{variant} f64 {m}x{n}: {rel:.3e}"
    np.testing.assert_allclose(f.beta, ref.beta, rtol=1e-12)
    assert abs(err - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)
