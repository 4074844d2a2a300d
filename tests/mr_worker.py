"""One rank of a multi-process test (launched by tests/test_multirank.py).

    RANK=r WORLD_SIZE=P MASTER_ADDR=127.0.0.1 MASTER_PORT=... python tests/mr_worker.py MODE OUT [args]

MODE
  solve     distributed_solve through the product (DistSession over the fused
            peer-memory exchange, or NCCL) on this rank's row block of
            gen_problem_t(seed, rows, cols); every rank may share one GPU.
  protocol  the per-iteration exchange protocol of distributed_solve
            (distributed.hpp:52-130) restated on the CPU with the oracle's
            row pass per rank and a real gloo all-gather of (column sums,
            alpha error) summed in ascending rank order — what the sessions do
            on device; checked against the oracle's distributed_solve.
  bytes     the host handshake helpers (all_gather_bytes / broadcast_bytes).
  io        every rank streams its row block of a .uotp file into its session,
            solves, and writes the plan back collectively (one shared file).
Results go to OUT/rank{r}.npz (or .json).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch.distributed as dist
    mode, out = sys.argv[1], sys.argv[2]
    args = [float(x) if "." in x or "e" in x else int(x) for x in sys.argv[3:]]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    try:
        if mode == "solve":
            solve(rank, world, out, *args)
        elif mode == "protocol":
            protocol(rank, world, out, *args)
        elif mode == "bytes":
            handshake(rank, world, out)
        elif mode == "io":
            io_roundtrip(rank, world, out, *args)
        else:
            raise SystemExit(f"unknown mode {mode}")
    finally:
        dist.barrier()
        dist.destroy_process_group()


def solve(rank, world, out, seed, rows, cols, k, tol, ep, balance=0):
    from paper_2412_11079_b200 import distributed as D
    from paper_2412_11079_b200 import uot
    exchange = os.environ.get("UOT_EXCHANGE", "peer")
    md = os.environ.get("MR_DEVICE", "0")
    device = rank if md == "rank" else int(md)  # "rank": one GPU per rank
    b, e = uot.RankPartition.make(world, rows).blocks[rank]
    p = uot.gen_block(seed, rows, cols, b, e - b)
    p.er, p.ep = 1.0, ep
    if balance:  # equal masses (test_fused.cpp:222-231): cpd scaled to sum(rpd)
        full = uot.gen_problem_t(seed, rows, cols)
        p.cpd = p.cpd * (full.rpd.sum() / p.cpd.sum())
    r = D.distributed_solve(p, tol, k, device=device, global_rows=rows, exchange=exchange)
    np.savez(os.path.join(out, f"rank{rank}.npz"), plan=r.plan, alpha=r.factors.alpha, beta=r.factors.beta,
             it=r.report.iterations, err=r.report.final_error, conv=r.report.converged,
             calls=r.comm.allreduce_calls, dbl=r.comm.doubles_reduced, b=b, e=e)


def protocol(rank, world, out, seed, rows, cols, k, ep):
    import torch
    import torch.distributed as dist

    import oracle
    o = oracle.Oracle()
    a, rpd, cpd = o.gen_problem(seed, rows, cols)
    b, e = o.rank_partition(world, rows)[rank:rank + 2]
    blk, rpd_b = np.ascontiguousarray(a[b:e]), rpd[b:e]
    fi = o.compute_fi(1.0, ep)

    def exchange(vec):  # one all-gather, then the ascending-rank sum (allreduce_vectors)
        parts = [torch.empty(vec.size, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(vec))
        acc = np.zeros(vec.size, np.float64)
        for q in range(world):
            acc += parts[q].numpy()
        return acc, parts

    cs, _ = exchange(o.init_col_sums(blk, 1))
    err = 0.0
    for _ in range(k):
        local = cs.copy()
        alpha, beta = o.fused_iterate(blk, local, rpd_b, cpd, fi, 1)  # beta from cs; local <- block partials
        ea = float(np.max(np.abs(alpha - 1.0)))
        vec = np.concatenate([local, np.zeros(world)])
        vec[cols + rank] = ea  # alpha error in this rank's slot
        red, _ = exchange(vec)
        cs = red[:cols]
        err = max(float(np.max(red[cols:])), float(np.max(np.abs(beta - 1.0))))
    np.savez(os.path.join(out, f"rank{rank}.npz"), plan=blk, alpha=alpha, beta=beta, err=err, b=b, e=e)


def io_roundtrip(rank, world, out, k):
    from paper_2412_11079_b200 import distributed as D
    from paper_2412_11079_b200 import uot
    src = os.environ["MR_UOTP"]
    info = uot.problem_file_info(src)
    s = D.make_session(info["m"], info["n"], int(os.environ.get("MR_DEVICE", "0")))
    try:
        s.load_problem_file(src)
        s.init_col_sums()
        it, err, conv = s.iterate(k, 1e-300)
        s.save_problem_file(os.path.join(out, "plan.uotp"))
        np.savez(os.path.join(out, f"rank{rank}.npz"), it=it, err=err, b=s.row_offset, e=s.row_offset + s.rows)
    finally:
        s.close()


def handshake(rank, world, out):
    from paper_2412_11079_b200 import distributed as D
    got = D.all_gather_bytes(bytes([rank]) * 64)
    bc = D.broadcast_bytes(b"id-of-rank-0" if rank == 0 else None, src=0)
    with open(os.path.join(out, f"rank{rank}.json"), "w") as f:
        json.dump({"gathered": [g.hex() for g in got], "bcast": bc.decode()}, f)


if __name__ == "__main__":
    main()
