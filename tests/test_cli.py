"""uot-cuda: the reference CLI's gen / solve / bench (tools/uot_main.cpp) on the
C ABI. CPU: gen writes the reference's container byte for byte, errors exit 1,
and solve has no CPU fallback. GPU: the JSON report and the written plan match
the oracle; exit codes follow uot_main.cpp (0 converged, 2 not)."""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

from conftest import KNEVER, ROOT, cuda_ok

CLI = os.path.join(ROOT, "paper_2412_11079_b200", "uot-cuda")


@pytest.fixture(scope="module")
def cli():
    from paper_2412_11079_b200 import build
    build.build()
    return build.build_cli()


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=300)


@pytest.mark.parametrize("dtype", ["fp32", "fp64"])
def test_gen_matches_reference_container(cli, orc, tmp_path, dtype):
    out = tmp_path / "g.uotp"
    r = run(cli, "gen", "--out", out, "--seed", 7, "--m", 5, "--n", 9, "--dtype", dtype)
    assert r.returncode == 0, r.stderr
    a, rpd, cpd = orc.gen_problem(7, 5, 9, dtype=np.float64 if dtype == "fp64" else np.float32)
    mine = tmp_path / "m.uotp"
    from paper_2412_11079_b200 import uot
    uot.write_problem(mine, uot.Problem(a, rpd, cpd, 1.0, 1.0))  # byte-identical to write_problem (test_io.py)
    assert out.read_bytes() == mine.read_bytes()


def test_usage_and_errors(cli, tmp_path):
    assert run(cli, "--help").returncode == 0
    assert run(cli).returncode == 1
    assert run(cli, "frobnicate").returncode == 1
    assert run(cli, "gen", "--m", 3).returncode == 1  # --out missing
    assert run(cli, "gen", "--out", tmp_path / "x", "--dtype", "fp16").returncode == 1


@pytest.mark.skipif(cuda_ok(), reason="checks the no-GPU behaviour")
def test_solve_without_gpu_fails_loudly(cli):
    r = run(cli, "solve", "--m", 8, "--n", 8)
    assert r.returncode == 1 and "error" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["fp32", "fp64"])
def test_solve_report_and_plan_match_oracle(gpu, cli, orc, tmp_path, dtype):
    src, plan_out, rep = tmp_path / "p.uotp", tmp_path / "plan.uotp", tmp_path / "r.json"
    assert run(cli, "gen", "--out", src, "--seed", 3, "--m", 300, "--n", 2000, "--dtype", dtype).returncode == 0
    r = run(cli, "solve", "--in", src, "--tol", KNEVER, "--max-iter", 12, "--out", rep, "--plan-out", plan_out)
    assert r.returncode == 2, r.stderr  # ran max_iter without converging
    d = json.load(open(rep))
    a, rpd, cpd = orc.gen_problem(3, 300, 2000, dtype=np.float64 if dtype == "fp64" else np.float32)
    ref = orc.fused_solve(a, rpd, cpd, 1.0, 1.0, KNEVER, 12, 1)
    assert d["solver"] == "cuda" and d["M"] == 300 and d["N"] == 2000 and d["dtype"] == dtype
    assert d["iterations"] == 12 and not d["converged"]
    assert abs(d["final_error"] - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)
    back = gpu.read_problem(plan_out)
    rel = np.max(np.abs(back.a.astype(np.float64) - ref.plan) / ref.plan)
    assert rel <= 1e-5


@pytest.mark.gpu
def test_solve_converges_with_exit_zero(gpu, cli, tmp_path):
    r = run(cli, "solve", "--seed", 4, "--m", 64, "--n", 64, "--dtype", "fp64", "--tol", 0.5, "--max-iter", 1000)
    d = json.loads(r.stdout)
    assert (r.returncode == 0) == d["converged"]


@pytest.mark.gpu
def test_bench_csv(gpu, cli):
    r = run(cli, "bench", "--sizes", "256,1024", "--solvers", "cuda,baseline,tiled", "--iters", 5)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "M,N,solver,workers,iterations,wall_ms,bytes_modeled"
    rows = [l.split(",") for l in lines[1:]]
    assert len(rows) == 6 and all(int(x[4]) == 5 and float(x[5]) > 0 for x in rows)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["fp32", "fp64"])
def test_solve_dist_matches_distributed_solve(gpu, cli, orc, tmp_path, dtype):
    # uot_main.cpp:109-111: --solver dist --ranks P -> distributed_solve(p, tol, max_iter, P)
    src, plan_out = tmp_path / "p.uotp", tmp_path / "plan.uotp"
    assert run(cli, "gen", "--out", src, "--seed", 6, "--m", 301, "--n", 3000, "--dtype", dtype).returncode == 0
    r = run(cli, "solve", "--in", src, "--solver", "dist", "--ranks", 3, "--devices", "0,0,0", "--tol", KNEVER,
            "--max-iter", 7, "--plan-out", plan_out)
    assert r.returncode == 2, r.stderr
    d = json.loads(r.stdout)
    assert d["solver"] == "dist" and d["ranks"] == 3 and d["iterations"] == 7 and d["dtype"] == dtype
    a, rpd, cpd = orc.gen_problem(6, 301, 3000, dtype=np.float64 if dtype == "fp64" else np.float32)
    if dtype == "fp32":
        ref = orc.distributed_solve(a, rpd, cpd, 1.0, 1.0, KNEVER, 7, 3)
    else:
        ref = orc.fused_solve(a, rpd, cpd, 1.0, 1.0, KNEVER, 7, 3)  # (= distributed_solve, test_distributed.cpp)
    assert abs(d["final_error"] - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)
    back = gpu.read_problem(plan_out)
    rel = np.max(np.abs(back.a.astype(np.float64) - ref.plan) / ref.plan)
    assert rel <= (1e-12 if dtype == "fp64" else 1e-5)
    # generated in HBM per rank, more ranks than rows -> PartitionError (exit 1)
    g = run(cli, "solve", "--seed", 2, "--m", 100, "--n", 500, "--dtype", dtype, "--solver", "dist", "--ranks", 2,
            "--devices", "0,0", "--max-iter", 3, "--tol", KNEVER)
    assert g.returncode == 2 and json.loads(g.stdout)["ranks"] == 2
    assert run(cli, "solve", "--m", 3, "--n", 8, "--solver", "dist", "--ranks", 4).returncode == 1


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [("fp64", None), ("fp32", 1e-6)])
def test_verify_every_solver_agrees_with_baseline(gpu, cli, dtype, tol):
    # uot_main.cpp:131-175: fused / parallel / tiled / dist vs baseline after --iters iterations
    args = ["verify", "--seed", 5, "--m", 130, "--n", 900, "--dtype", dtype, "--iters", 12, "--ranks", 3]
    if tol is not None:
        args += ["--tol", tol]
    r = run(cli, *args)
    d = json.loads(r.stdout)
    assert set(d) == {"iterations", "workers", "ranks", "diff_vs_baseline", "max_diff", "tolerance", "ok"}
    assert set(d["diff_vs_baseline"]) == {"fused", "parallel", "tiled", "dist"}
    assert d["iterations"] == 12 and d["ranks"] == 3 and d["ok"] and r.returncode == 0, r.stdout + r.stderr
    assert d["max_diff"] <= (1e-10 if dtype == "fp64" else 1e-6)
    bad = run(cli, "verify", "--seed", 5, "--m", 130, "--n", 900, "--dtype", dtype, "--iters", 3, "--tol", -1)
    assert bad.returncode == 2 and not json.loads(bad.stdout)["ok"]  # tolerance not met -> exit 2
