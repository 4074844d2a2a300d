"""Multi-rank (row-sharded) path: distributed_solve, distributed.hpp:52-136.

CPU (gloo, world size 2 and 3): the host handshake the sessions use, and the
per-iteration exchange protocol (column sums + alpha error, ascending-rank sum)
restated on the oracle's row pass, checked bitwise against the oracle's
distributed_solve. GPU: two ranks as two processes sharing one B200, their
column sums combined by the fused peer-memory exchange (CUDA IPC) inside the
finalize kernels, checked against the oracle's distributed_solve
(test_distributed.cpp:106-118: distributed == fused with P workers).
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import KNEVER, ROOT

WORKER = os.path.join(ROOT, "tests", "mr_worker.py")


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_ranks(world: int, mode: str, out: str, *args, env_extra=None, timeout=300):
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **(env_extra or {}))
        procs.append(subprocess.Popen([sys.executable, WORKER, mode, out, *map(str, args)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(o)
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r]}"
    return logs


# ------------------------------------------------------------------ CPU --

@pytest.mark.parametrize("world", [2, 3])
def test_handshake_helpers(tmp_path, world):
    run_ranks(world, "bytes", str(tmp_path))
    for r in range(world):
        d = json.load(open(tmp_path / f"rank{r}.json"))
        assert d["gathered"] == [(bytes([q]) * 64).hex() for q in range(world)]
        assert d["bcast"] == "id-of-rank-0"


@pytest.mark.parametrize("world,rows,cols,k", [(2, 37, 50, 12), (3, 64, 33, 9)])
def test_exchange_protocol_matches_reference(tmp_path, orc, world, rows, cols, k):
    run_ranks(world, "protocol", str(tmp_path), 7, rows, cols, k, 0.1)
    a, rpd, cpd = orc.gen_problem(7, rows, cols)
    ref = orc.distributed_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, world)
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        b, e = int(d["b"]), int(d["e"])
        assert np.array_equal(d["plan"], ref.plan[b:e])
        assert np.array_equal(d["alpha"], ref.alpha[b:e])
        assert np.array_equal(d["beta"], ref.beta)
        assert float(d["err"]) == ref.final_error


# ------------------------------------------------------------------ GPU --

def _check_solve(tmp_path, orc, world, rows, cols, k, tol, ep, seed=42, balance=False):
    a, rpd, cpd = orc.gen_problem(seed, rows, cols)
    if balance:
        cpd = cpd * (rpd.sum() / cpd.sum())
    ref = orc.distributed_solve(a, rpd, cpd, 1.0, ep, tol, k, world)
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        b, e = int(d["b"]), int(d["e"])
        assert int(d["it"]) == ref.iterations
        plan = d["plan"]
        rel = np.max(np.abs(plan.astype(np.float64) - ref.plan[b:e]) / ref.plan[b:e])
        assert rel <= 1e-5, f"rank {r}: max rel err {rel:.3e}"
        np.testing.assert_allclose(d["alpha"], ref.alpha[b:e], rtol=1e-12)
        np.testing.assert_allclose(d["beta"], ref.beta, rtol=1e-12)
        assert abs(float(d["err"]) - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)
        assert int(d["calls"]) == int(d["it"])
    # every rank derived the identical beta from the identical exchanged sums
    betas = [np.load(tmp_path / f"rank{r}.npz")["beta"] for r in range(world)]
    assert all(np.array_equal(betas[0], x) for x in betas[1:])


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,k", [(300, 2000, 10), (64, 20000, 6)])  # G == 1 and G > 1 sweeps
def test_two_ranks_one_gpu_peer_exchange(gpu, orc, tmp_path, rows, cols, k):
    run_ranks(2, "solve", str(tmp_path), 42, rows, cols, k, KNEVER, 0.1,
              env_extra={"UOT_EXCHANGE": "peer", "MR_DEVICE": "0"})
    _check_solve(tmp_path, orc, 2, rows, cols, k, KNEVER, 0.1)


@pytest.mark.gpu
def test_two_ranks_converge_at_the_same_iteration(gpu, orc, tmp_path):
    # early exit on the exchanged error: both ranks stop where distributed_solve stops
    run_ranks(2, "solve", str(tmp_path), 5, 300, 9000, 10000, 1e-6, 0.0, 1,
              env_extra={"UOT_EXCHANGE": "peer", "MR_DEVICE": "0"})
    _check_solve(tmp_path, orc, 2, 300, 9000, 10000, 1e-6, 0.0, seed=5, balance=True)
    for r in range(2):
        assert bool(np.load(tmp_path / f"rank{r}.npz")["conv"])


@pytest.mark.gpu
def test_three_ranks_one_gpu_peer_exchange(gpu, orc, tmp_path):
    run_ranks(3, "solve", str(tmp_path), 3, 257, 1000, 8, KNEVER, 0.1,
              env_extra={"UOT_EXCHANGE": "peer", "MR_DEVICE": "0"})
    _check_solve(tmp_path, orc, 3, 257, 1000, 8, KNEVER, 0.1, seed=3)


# ------------------------------------------------ NCCL / cross-device paths --

def _ngpus() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except ImportError:
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,k", [(300, 2000, 10), (64, 20000, 6)])
def test_single_rank_nccl_exchange_path(gpu, orc, rows, cols, k):
    """uot_create_dist with one rank and an NCCL id runs the NCCL exchange path
    (stage-1 reduce -> ncclAllReduce over a one-rank communicator -> stage-2
    beta, allreduce.cpp:6-15 with P = 1) on one GPU; == distributed_solve(1)."""
    from paper_2412_11079_b200 import distributed as D
    a, rpd, cpd = orc.gen_problem(42, rows, cols)
    ref = orc.distributed_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, k, 1)
    s = D.DistSession(rows, cols, 0, 1, 0, D.nccl_unique_id(), "nccl")
    try:
        assert s.exchange_mode() == 1 and s.layout["resident"] == 0
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.1))
        s.init_col_sums()
        it, err, conv = s.iterate(k, KNEVER)
        f = s.factors()
        plan = s.plan()
        calls, dbl = s.comm_stats()
    finally:
        s.close()
    assert it == k and calls == k and dbl == k * cols
    rel = np.max(np.abs(plan.astype(np.float64) - ref.plan) / ref.plan)
    assert rel <= 1e-5
    np.testing.assert_allclose(f.beta, ref.beta, rtol=1e-12)
    np.testing.assert_allclose(f.alpha, ref.alpha, rtol=1e-12)
    assert abs(err - ref.final_error) <= 1e-9 * max(1.0, ref.final_error)


@pytest.mark.gpu
def test_single_rank_nccl_early_exit(gpu, orc):
    from paper_2412_11079_b200 import distributed as D
    a, rpd, cpd = orc.gen_problem(5, 200, 3000)
    cpd = cpd * (rpd.sum() / cpd.sum())
    ref = orc.distributed_solve(a, rpd, cpd, 1.0, 0.0, 1e-6, 10000, 1)
    s = D.DistSession(200, 3000, 0, 1, 0, D.nccl_unique_id(), "nccl")
    try:
        s.set_problem(gpu.Problem(a, rpd, cpd, 1.0, 0.0))
        s.init_col_sums()
        it, err, conv = s.iterate(10000, 1e-6)
    finally:
        s.close()
    assert ref.converged and conv and it == ref.iterations


@pytest.mark.gpu
@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (gpurun and the round-end box have one)")
@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_two_ranks_two_gpus(gpu, orc, tmp_path, exchange):
    """One process per GPU: the peer exchange over NVLink (CUDA IPC across
    devices, st.release.sys / ld.acquire.sys flags) and a real 2-rank NCCL
    allreduce, both == distributed_solve(2)."""
    run_ranks(2, "solve", str(tmp_path), 42, 300, 20000, 8, KNEVER, 0.1,
              env_extra={"UOT_EXCHANGE": exchange, "MR_DEVICE": "rank", "UOT_EXCHANGE_FALLBACK": "0"})
    _check_solve(tmp_path, orc, 2, 300, 20000, 8, KNEVER, 0.1)


@pytest.mark.gpu
@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (gpurun and the round-end box have one)")
def test_in_process_group_over_distinct_gpus(gpu, orc):
    """uot_create_group with rank r on GPU r: peer access + direct remote stores
    across devices, == distributed_solve(P)."""
    n = min(_ngpus(), 4)
    a, rpd, cpd = orc.gen_problem(9, 600, 20000)
    ref = orc.distributed_solve(a, rpd, cpd, 1.0, 0.1, KNEVER, 7, n)
    res = gpu.distributed_solve(gpu.Problem(a, rpd, cpd, 1.0, 0.1), KNEVER, 7, n, devices=list(range(n)))
    rel = np.max(np.abs(res.plan.astype(np.float64) - ref.plan) / ref.plan)
    assert rel <= 1e-5 and res.report.iterations == 7
    np.testing.assert_allclose(res.factors.beta, ref.beta, rtol=1e-12)
