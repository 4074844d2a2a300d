"""Multi-GPU row-sharded solve: one process per GPU, one allreduce per iteration.

Mirror of distributed_solve (/root/reference/proj/core/include/uot/distributed.hpp:52-136).
The reference simulates P ranks in one process; here each rank is a process
driving its own B200:

* rows are split by RankPartition::make(P, rows) (src/plan.cpp:35-44) — rank r
  keeps its contiguous row block resident in HBM;
* every iteration ends with ONE exchange of the ranks' column partials
  (distributed.hpp:88-94) plus each rank's max|alpha-1| (the "scalar
  max-reduction" the reference comment at distributed.hpp:50-51 anticipates,
  folded into the same exchange), either fused into the finalize kernels over
  peer memory (default: CUDA IPC over NVLink/NVSwitch, ascending-rank sum =
  allreduce_vectors, src/allreduce.cpp:6-15) or as one ncclAllReduce;
* every rank then derives the identical beta from the identical reduced vector
  (distributed.hpp:96-100).

The peer mappings / NCCL communicator live inside the C++ session
(include/uot_cuda.h, uot_create_peer / uot_create_dist); torch.distributed (any
backend, gloo is enough) only carries the 64-byte IPC handles (or the 128-byte
NCCL id of rank 0) and the host-side barriers.
"""
from __future__ import annotations

import ctypes as C
import os
import time
import warnings

from . import uot


# CommStats / DistributedResult (distributed.hpp:24-40) are shared with the
# in-process uot.distributed_solve; here a result holds THIS rank's row block.
CommStats = uot.CommStats
DistributedResult = uot.DistributedResult


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = uot.lib().uot_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc:
        raise uot.CudaError("ncclGetUniqueId failed (libnccl.so.2 missing?)")
    return bytes(buf)


def _torch_dist():
    import torch.distributed as dist  # plumbing only
    if not dist.is_available() or not dist.is_initialized():
        return None
    return dist


def broadcast_bytes(data: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string over the initialised torch process group."""
    dist = _torch_dist()
    if dist is None:
        assert data is not None
        return data
    obj = [data]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def rank_block(ranks: int, rows: int, rank: int):
    part = uot.RankPartition.make(ranks, rows)
    return part.blocks[rank]


class DistSession(uot.Session):
    """Session for rank `rank` of `nranks` over `global_rows` rows. With
    nranks == 1 it is an ordinary single-GPU session (no exchange).

    exchange="peer" (default): the per-iteration allreduce is fused into the
    finalize kernels over peer memory (CUDA IPC over NVLink/NVSwitch; see
    csrc/finalize.cuh) — call connect() with every rank's handle() before use.
    exchange="nccl": one ncclAllReduce per iteration (needs the NCCL id of rank 0).
    """

    def __init__(self, global_rows: int, cols: int, rank: int, nranks: int, device: int,
                 nccl_id: bytes | None = None, exchange: str = "peer"):
        if exchange not in ("peer", "nccl"):
            raise uot.InvalidParameter(f"exchange must be 'peer' or 'nccl', not {exchange!r}")
        if exchange == "nccl" and nranks > 1 and nccl_id is None:
            raise uot.InvalidParameter("a multi-rank NCCL session needs the NCCL id of rank 0")
        dist = (rank, nranks, "peer") if exchange == "peer" else (rank, nranks, nccl_id)
        super().__init__(global_rows, cols, device, dist=dist)
        self.rank, self.nranks, self.exchange = rank, nranks, exchange

    def handle(self) -> bytes:
        """The 64-byte CUDA IPC handle of this rank's exchange region."""
        buf = (C.c_uint8 * 64)()
        self._check(uot.lib().uot_peer_handle(self._h, C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def connect(self, handles: list[bytes]):
        """Map every rank's exchange region (handles in rank order; own included)."""
        if len(handles) != self.nranks or any(len(h) != 64 for h in handles):
            raise uot.InvalidParameter(f"connect needs {self.nranks} handles of 64 bytes")
        buf = (C.c_uint8 * (64 * self.nranks)).from_buffer_copy(b"".join(handles))
        self._check(uot.lib().uot_peer_connect(self._h, C.cast(buf, C.c_void_p)))

    def exchange_mode(self) -> int:
        return int(uot.lib().uot_exchange_mode(self._h))


def all_gather_bytes(data: bytes) -> list[bytes]:
    """Every rank's byte string, in rank order, over the torch process group."""
    dist = _torch_dist()
    if dist is None:
        return [data]
    out: list = [None] * dist.get_world_size()
    dist.all_gather_object(out, data)
    return out


def make_session(global_rows: int, cols: int, device: int | None = None,
                 exchange: str | None = None) -> DistSession:
    """Collective: one DistSession per rank of the current torch process group.
    The exchange defaults to $UOT_EXCHANGE or "peer"."""
    dist = _torch_dist()
    rank = dist.get_rank() if dist else 0
    world = dist.get_world_size() if dist else 1
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", rank))
    exchange = exchange or os.environ.get("UOT_EXCHANGE", "peer")
    if world > 1 and exchange == "peer":
        s = DistSession(global_rows, cols, rank, world, device, None, "peer")
        why = _connect_peers(s)
        if why is None:
            return s
        s.close()
        # Every rank saw the same verdict (all-gathered), so all fall back together.
        if os.environ.get("UOT_EXCHANGE_FALLBACK", "1") == "0":
            raise uot.CudaError(f"peer exchange unavailable: {why}")
        warnings.warn(f"peer exchange unavailable ({why}); using one NCCL allreduce per iteration")
        exchange = "nccl"
    nid = None
    if world > 1 and exchange == "nccl":
        nid = broadcast_bytes(nccl_unique_id() if rank == 0 else None, src=0)
    return DistSession(global_rows, cols, rank, world, device, nid, exchange)


def _connect_peers(s: DistSession) -> str | None:
    """Collective: exchange the IPC handles and map every peer's region. Returns
    None when every rank connected, else the first failure (same on all ranks)."""
    try:
        h = s.handle()
    except uot.Error as e:
        h = b"!" + str(e).encode()[:200]
    handles = all_gather_bytes(h)
    bad = [x for x in handles if len(x) != 64]
    err = b""
    if bad:
        err = bad[0][1:]
    else:
        try:
            s.connect(handles)
        except uot.Error as e:
            err = str(e).encode()[:200] or b"connect failed"
    errs = [e for e in all_gather_bytes(err) if e]
    return errs[0].decode(errors="replace") if errs else None


def distributed_solve(p: uot.Problem, tol: float, max_iter: int, device: int | None = None,
                      session: DistSession | None = None, global_rows: int | None = None,
                      exchange: str | None = None) -> DistributedResult:
    """distributed_solve (distributed.hpp:52-130) across the ranks of the current
    torch process group (world size 1 without one).

    `p` is the whole problem (every rank slices its RankPartition block), or —
    with `global_rows` given — already this rank's row block (rpd of the block,
    cpd of all columns), which avoids materialising the global matrix per host."""
    uot._validate_controls(tol, max_iter, "distributed_solve")
    t0 = time.perf_counter()
    grows = global_rows if global_rows is not None else p.m()
    own = session is None
    s = make_session(grows, p.n(), device, exchange) if own else session
    try:
        b, e = s.row_offset, s.row_offset + s.rows
        if global_rows is None:
            local = uot.Problem(p.a[b:e], p.rpd[b:e], p.cpd, p.er, p.ep)
        else:
            if p.m() != s.rows:
                raise uot.PartitionError(f"rank block has {p.m()} rows, partition expects {s.rows}")
            local = p
        s.set_problem(local)
        s.init_col_sums()
        it, err, conv = s.iterate(max_iter, tol)
        f = s.factors()
        plan = s.plan()
        calls, dbl = s.comm_stats()
    finally:
        if own:
            s.close()
    rep = uot.SolveReport("dist", it, err, conv, (time.perf_counter() - t0) * 1e3)
    return DistributedResult(plan, f, rep, CommStats(calls, dbl), b, e)
