"""Parity at the BASELINE configurations' FULL sizes and iteration counts:
the GPU's fused_solve against the reference's own fused_solve (oracle/_ref:
the reference compiled from its sources; the C restatement if absent), both
from the same gen_problem_t<float>(42, R, C) with er = 1, ep = 0.1.

Test infrastructure (it runs the checker), not a bench: the CPU leg is the
reference's threaded fused_iterate_parallel over all host cores.

python tools/full_parity.py [--only 1,2,3,4,5] [--f64] [--json OUT]
(--f64: Problem<double> of the same shapes; tolerance 1e-12 instead of 1e-5)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2412_11079_b200 import uot  # noqa: E402

# (config, rows, cols, K, ranks): config 5 runs as 4 in-process ranks (one GPU here) against the
# reference's fused_solve with 4 workers, which is bitwise its distributed_solve(4)
# (test_distributed.cpp:106-118); K = 20 keeps the 4-thread CPU leg near two minutes
CONFIGS = [(1, 1024, 1024, 100, 1), (2, 8192, 8192, 500, 1), (3, 32768, 32768, 200, 1),
           (4, 262144, 4096, 200, 1), (5, 131072, 32768, 20, 4)]
only = None
if "--only" in sys.argv:
    only = {int(x) for x in sys.argv[sys.argv.index("--only") + 1].split(",")}
ref = oracle.RefOracle() if oracle.have_ref() else oracle.Oracle()
kind = "reference (oracle/_ref)" if isinstance(ref, oracle.RefOracle) else "C restatement (oracle/uot_oracle.c)"
gen = oracle.Oracle()
threads = os.cpu_count() or 1


def max_rel(x, y, chunk=1 << 24):  # chunked: no full-size float64 temporaries
    xf, yf = x.reshape(-1), y.reshape(-1)
    m = 0.0
    for i in range(0, xf.size, chunk):
        a64, b64 = xf[i:i + chunk].astype(np.float64), yf[i:i + chunk].astype(np.float64)
        m = max(m, float(np.max(np.abs(a64 - b64) / b64)))
    return m


F64 = "--f64" in sys.argv
DT = np.float64 if F64 else np.float32
BAR = 1e-12 if F64 else 1e-5
rows = []
for idx, m, n, k, ranks in CONFIGS:
    if only and idx not in only:
        continue
    a, rpd, cpd = gen.gen_problem(42, m, n, dtype=DT, threads=threads)
    workers = threads if ranks == 1 else ranks
    t0 = time.time()
    r = ref.fused_solve(a, rpd, cpd, 1.0, 0.1, 1e-300, k, workers)
    t_cpu = time.time() - t0
    t0 = time.time()
    p = uot.Problem(a, rpd, cpd, 1.0, 0.1)
    g = uot.fused_solve(p, 1e-300, k) if ranks == 1 else uot.distributed_solve(p, 1e-300, k, ranks, devices=[0] * ranks)
    t_gpu = time.time() - t0
    row = {
        "config": idx, "rows": m, "cols": n, "iterations": k, "ranks": ranks, "checker": kind,
        "dtype": "f64" if F64 else "f32",
        "cpu_threads": workers, "iterations_gpu": g.report.iterations, "iterations_ref": r.iterations,
        "plan_max_rel_err": max_rel(g.plan, r.plan),
        "plan_bitwise_equal_fraction": float(np.mean(g.plan == r.plan)),
        "alpha_max_rel_err": float(np.max(np.abs(g.factors.alpha - r.alpha) / r.alpha)),
        "beta_max_rel_err": float(np.max(np.abs(g.factors.beta - r.beta) / r.beta)),
        "final_error_gpu": g.report.final_error, "final_error_ref": r.final_error,
        "row_marginal_err_gpu": float(np.max(np.abs(g.plan.sum(1, dtype=np.float64) - rpd) / rpd)),
        "row_marginal_err_ref": float(np.max(np.abs(r.plan.sum(1, dtype=np.float64) - rpd) / rpd)),
        "col_marginal_err_gpu": float(np.max(np.abs(g.plan.sum(0, dtype=np.float64) - cpd) / cpd)),
        "col_marginal_err_ref": float(np.max(np.abs(r.plan.sum(0, dtype=np.float64) - cpd) / cpd)),
        "wall_s_ref": t_cpu, "wall_s_gpu_incl_pcie": t_gpu,
    }
    ok = row["plan_max_rel_err"] <= BAR and row["iterations_gpu"] == row["iterations_ref"]
    row["within_bar"] = bool(ok)
    row["bar"] = BAR
    rows.append(row)
    print(f"config {idx} {m}x{n} {row['dtype']} K={k} ranks={ranks}: plan max rel {row['plan_max_rel_err']:.2e}, bitwise "
          f"{row['plan_bitwise_equal_fraction'] * 100:.4f}%, alpha {row['alpha_max_rel_err']:.1e}, beta "
          f"{row['beta_max_rel_err']:.1e}, err {row['final_error_gpu']:.6e} vs {row['final_error_ref']:.6e} "
          f"[{kind}, {workers} threads: {t_cpu:.1f} s; GPU incl. PCIe {t_gpu:.2f} s] {'OK' if ok else 'FAIL'}",
          flush=True)
    del a, r, g
if "--json" in sys.argv:
    json.dump(rows, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
sys.exit(0 if all(r["within_bar"] for r in rows) else 1)
