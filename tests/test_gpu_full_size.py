"""Parity at the BASELINE configurations' FULL sizes and iteration counts,
against the reference itself (oracle/_ref: the unmodified reference compiled
from its sources) — the north_star bar: max relative error <= 1e-5 on P and on
both marginal errors after K iterations, same inputs (gen_problem_t<float>(42),
er = 1, ep = 0.1).

* config 3 (32768 x 32768, K = 200) and config 4 (262144 x 4096, K = 200):
  uot.Session vs the reference's fused_iterate_parallel loop at W = nproc
  (fused_solve's loop, fused.hpp:259-285, without the stop test);
* config 5 (131072 x 32768, row-sharded, K = 20): the in-process rank group
  (uot_create_group, distributed_solve's own call shape, distributed.hpp:52-142)
  with 2 and 4 ranks — on distinct GPUs when the box has them, else sharing
  GPU 0 — against the reference's W-worker iteration at W = nproc (its
  distributed_solve(W) is bitwise the same, test_distributed.cpp:106-118).

The GPU generates the problem in HBM (bit-identical to gen_problem_t, tested in
test_gpu_parity.py) and the plans are compared block by block, so the host
holds at most two copies of a config-5 matrix.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import KNEVER

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-5
ER, EP = 1.0, 0.1
THREADS = os.cpu_count() or 1


class Compare:
    """Accumulates P error, bitwise fraction and both marginals block by block."""

    def __init__(self, ref_plan, rpd, cpd):
        self.ref, self.rpd, self.cpd = ref_plan, rpd, cpd
        n = ref_plan.shape[1]
        self.max_rel, self.equal, self.count = 0.0, 0, 0
        self.row_err_g, self.row_err_r = 0.0, 0.0
        self.col_g, self.col_r = np.zeros(n), np.zeros(n)

    def block(self, r0, plan_block, step=2048):
        for i in range(0, plan_block.shape[0], step):
            g = plan_block[i:i + step]
            r = self.ref[r0 + i:r0 + i + g.shape[0]]
            g64, r64 = g.astype(np.float64), r.astype(np.float64)
            self.max_rel = max(self.max_rel, float(np.max(np.abs(g64 - r64) / np.abs(r64))))
            self.equal += int(np.count_nonzero(g == r))
            self.count += g.size
            rp = self.rpd[r0 + i:r0 + i + g.shape[0]]
            self.row_err_g = max(self.row_err_g, float(np.max(np.abs(g64.sum(1) - rp))))
            self.row_err_r = max(self.row_err_r, float(np.max(np.abs(r64.sum(1) - rp))))
            self.col_g += g64.sum(0)
            self.col_r += r64.sum(0)

    def check(self, what):
        ec_g = float(np.max(np.abs(self.col_g - self.cpd)))
        ec_r = float(np.max(np.abs(self.col_r - self.cpd)))
        print(f"{what}: P max rel {self.max_rel:.2e}, bitwise {100.0 * self.equal / self.count:.5f}%, "
              f"row marginal err {self.row_err_g:.9e} vs {self.row_err_r:.9e}, "
              f"col marginal err {ec_g:.9e} vs {ec_r:.9e}")
        assert self.count == self.ref.size
        assert self.max_rel <= TOL, f"{what}: max rel err on P {self.max_rel:.3e}"
        assert abs(self.row_err_g - self.row_err_r) <= TOL * self.row_err_r, f"{what}: row marginal error"
        assert abs(ec_g - ec_r) <= TOL * ec_r, f"{what}: col marginal error"


def reference_run(ref, orc, m, n, k, workers):
    a, rpd, cpd = orc.gen_problem(42, m, n, threads=THREADS)
    out = ref.fused_iterate_k_inplace(a, rpd, cpd, ER, EP, workers, k)  # a <- the reference's plan
    return out, rpd, cpd


@pytest.mark.parametrize("cfg,m,n,k", [(3, 32768, 32768, 200), (4, 262144, 4096, 200)])
def test_baseline_config_full_k_vs_reference(gpu, orc, ref, cfg, m, n, k):
    r, rpd, cpd = reference_run(ref, orc, m, n, k, THREADS)
    with gpu.Session(m, n) as s:
        s.generate_problem(42, ER, EP)
        s.init_col_sums()
        it, err, conv = s.iterate(k, KNEVER)
        assert it == k and not conv
        f = s.factors()
        cmp = Compare(r.plan, rpd, cpd)
        cmp.block(0, s.plan())
    cmp.check(f"config {cfg} {m}x{n} K={k} vs the reference (W={THREADS})")
    np.testing.assert_allclose(f.alpha, r.alpha, rtol=1e-9)
    np.testing.assert_allclose(f.beta, r.beta, rtol=1e-9)
    assert abs(err - r.final_error) <= TOL * r.final_error


def _devices(ranks):
    import torch
    n = max(1, torch.cuda.device_count() if torch.cuda.is_available() else 1)
    return [r % n for r in range(ranks)]


def test_config5_row_sharded_ranks_vs_reference(gpu, orc, ref):
    m, n, k = 131072, 32768, 20
    r, rpd, cpd = reference_run(ref, orc, m, n, k, THREADS)  # == the reference's distributed_solve(THREADS)
    for ranks in (2, 4):
        with gpu.SessionGroup(m, n, ranks, devices=_devices(ranks)) as g:
            for s in g.ranks:
                s.generate_problem(42, ER, EP)
            g.init_col_sums()
            it, err, conv = g.iterate(k, KNEVER)
            assert it == k and not conv
            cmp = Compare(r.plan, rpd, cpd)
            alpha = np.empty(m)
            for s in g.ranks:
                b = s.row_offset
                f = s.factors()
                alpha[b:b + s.rows] = f.alpha
                cmp.block(b, s.plan())
                np.testing.assert_allclose(f.beta, r.beta, rtol=1e-9)
        cmp.check(f"config 5 {m}x{n} K={k} as {ranks} ranks on devices {_devices(ranks)} vs the reference "
                  f"(W={THREADS})")
        np.testing.assert_allclose(alpha, r.alpha, rtol=1e-9)
        assert abs(err - r.final_error) <= TOL * r.final_error
