"""Python mirror of the reference solver API (namespace uot), backed by the
sm_100a extension through its C ABI (include/uot_cuda.h).

Names, argument meaning and errors follow /root/reference/proj/core/include/uot:

  ==========================  =============================================
  here                        reference
  ==========================  =============================================
  Problem                     Problem<T>            problem.hpp:19-28
  ScalingFactors              ScalingFactors        problem.hpp:30-33
  SolveReport / SolveResult   problem.hpp:35-48
  FusedState                  FusedState            fused.hpp:19-23
  RankPartition.make          RankPartition::make   plan.cpp:35-44
  compute_fi / rescale_factor / convergence_error   scaling.cpp:9-29
  gen_problem_t               problem_io.hpp:17-31
  init_col_sums               fused.hpp:96-110
  fused_iterate               fused.hpp:164-191 / 197-250
  fused_solve                 fused.hpp:259-291
  Session                     (device-resident form of the loop above)
  read_problem / write_problem, Session.load_problem_file / save_problem_file
                              problem_io.cpp:13-141 (.uotp)
  Error, InvalidParameter, DegenerateSum, ConfigError, PartitionError, IoError
                              error.hpp:9-37
  ==========================  =============================================

There is no CPU fallback: importing this module without the built extension,
or using it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import build as _build

# ----------------------------------------------------------------- errors --


class Error(RuntimeError):
    """uot::Error (error.hpp:9-12)."""


class InvalidParameter(Error):
    """uot::InvalidParameter (error.hpp:14-17)."""


class DegenerateSum(Error):
    """uot::DegenerateSum (error.hpp:19-23)."""


class PartitionError(Error):
    """uot::PartitionError (error.hpp:29-32)."""


class ConfigError(Error):
    """uot::ConfigError (error.hpp:24-27): the launch cannot cover the matrix."""


class CudaError(Error):
    """CUDA / NCCL runtime failure (no reference analogue)."""


class IoError(Error):
    """uot::IoError (error.hpp:34-37): malformed or unreadable problem file."""


class CudaExtensionMissing(ImportError):
    """The sm_100a extension is not built; there is deliberately no fallback."""


_ERRORS = {1: InvalidParameter, 2: DegenerateSum, 3: PartitionError, 4: ConfigError,
           5: CudaError, 6: CudaError, 7: IoError}

UOT_F32, UOT_F64 = 1, 2

# ---------------------------------------------------------------- library --


class Layout(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("row_offset", C.c_uint64),
                ("global_rows", C.c_uint64), ("pitch", C.c_uint32), ("slice", C.c_uint32),
                ("G", C.c_uint32), ("groups", C.c_uint32), ("rows_per_step", C.c_uint32),
                ("threads", C.c_uint32), ("chunks", C.c_uint32), ("smem_bytes", C.c_uint32),
                ("nbuf", C.c_uint32), ("sms", C.c_uint32), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("device", C.c_int32), ("evict_first", C.c_int32),
                ("smid_map", C.c_int32), ("exchange", C.c_int32),
                ("resident", C.c_int32), ("dtype", C.c_int32),
                ("dynamic", C.c_int32), ("schedule", C.c_int32), ("pinned", C.c_int32),
                ("variant", C.c_int32), ("keep_batches", C.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_P = C.c_void_p
_u64, _d, _i = C.c_uint64, C.c_double, C.c_int


def lib():
    """Load libuot_cuda.so (built in-tree). Raises CudaExtensionMissing if absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("UOT_LIB_PATH") or _build.SO  # UOT_LIB_PATH: e.g. the trace build
    if not os.path.exists(path):
        if os.environ.get("UOT_AUTOBUILD", "1") == "1":
            try:
                _build.build()
            except Exception as e:  # noqa: BLE001
                raise CudaExtensionMissing(f"building {path} failed: {e}") from e
        else:
            raise CudaExtensionMissing(f"{path} is not built (python -m paper_2412_11079_b200.build)")
    L = C.CDLL(path)
    L.uot_create.argtypes = [C.POINTER(_P), _u64, _u64, _i, _i]
    L.uot_create_dist.argtypes = [C.POINTER(_P), _u64, _u64, _i, _i, _i, _i, _P]
    L.uot_nccl_unique_id.argtypes = [_P]
    L.uot_create_peer.argtypes = [C.POINTER(_P), _u64, _u64, _i, _i, _i, _i]
    L.uot_peer_handle.argtypes = [_P, _P]
    L.uot_peer_connect.argtypes = [_P, _P]
    L.uot_exchange_mode.argtypes = [_P]
    L.uot_create_group.argtypes = [_P, _u64, _u64, _i, _P, _i, _P]
    L.uot_group_init_col_sums.argtypes = [_P, _i]
    L.uot_group_iterate.argtypes = [_P, _i, _u64, _d, C.POINTER(_u64), C.POINTER(_d), C.POINTER(_i)]
    L.uot_set_variant.argtypes = [_P, _i]
    L.uot_set_deterministic.argtypes = [_P, _i]
    L.uot_set_resident.argtypes = [_P, _i]
    L.uot_set_schedule.argtypes = [_P, _i]
    L.uot_get_schedule_stats.argtypes = [_P, _P, _P, _P]
    L.uot_set_group_weights.argtypes = [_P, _P, C.c_uint32]
    L.uot_get_group_weights.argtypes = [_P, _P, C.c_uint32]
    L.uot_calibrate_schedule.argtypes = [_P, C.c_uint32]
    L.uot_problem_file_info.argtypes = [C.c_char_p, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_i),
                                        C.POINTER(_d), C.POINTER(_d)]
    L.uot_last_io_error.restype = C.c_char_p
    L.uot_load_problem_file.argtypes = [_P, C.c_char_p]
    L.uot_save_problem_file.argtypes = [_P, C.c_char_p]
    L.uot_destroy.argtypes = [_P]
    L.uot_destroy.restype = None
    L.uot_last_error.argtypes = [_P]
    L.uot_last_error.restype = C.c_char_p
    L.uot_get_layout.argtypes = [_P, C.POINTER(Layout)]
    L.uot_get_stream.argtypes = [_P]
    L.uot_get_stream.restype = _P
    L.uot_set_problem.argtypes = [_P, _P, _P, _P, _d, _d]
    L.uot_set_problem_f64.argtypes = [_P, _P, _P, _P, _d, _d]
    L.uot_set_plan_f64.argtypes = [_P, _P]
    L.uot_get_plan_f64.argtypes = [_P, _P]
    L.uot_gen_block_f64.argtypes = [_u64, _u64, _u64, _u64, _u64, _P, _P, _P, _i]
    L.uot_generate_problem.argtypes = [_P, _u64, _d, _d]
    L.uot_set_plan.argtypes = [_P, _P]
    L.uot_set_iterate_input.argtypes = [_P, _P, _i, _P, _P, _d]
    L.uot_set_fi.argtypes = [_P, _d]
    L.uot_init_col_sums.argtypes = [_P]
    L.uot_set_col_sums.argtypes = [_P, _P]
    L.uot_get_col_sums.argtypes = [_P, _P]
    L.uot_iterate.argtypes = [_P, _u64, _d, C.POINTER(_u64), C.POINTER(_d), C.POINTER(_i)]
    L.uot_iterate_timed.argtypes = [_P, _u64, _d, C.POINTER(_u64), C.POINTER(_d), C.POINTER(_i),
                                    C.POINTER(_d)]
    L.uot_synchronize.argtypes = [_P]
    L.uot_get_factors.argtypes = [_P, _P, _P]
    L.uot_get_plan.argtypes = [_P, _P]
    L.uot_get_report.argtypes = [_P, C.POINTER(_u64), C.POINTER(_d), C.POINTER(_i)]
    L.uot_get_comm_stats.argtypes = [_P, C.POINTER(_u64), C.POINTER(_u64)]
    L.uot_set_timing.argtypes = [_P, _i]
    L.uot_get_timing.argtypes = [_P, C.POINTER(_d), C.POINTER(_d), C.POINTER(_u64)]
    L.uot_kernel_launches.argtypes = [_P]
    L.uot_kernel_launches.restype = _u64
    L.uot_compute_fi.argtypes = [_d, _d, C.POINTER(_d)]
    L.uot_rescale_factor.argtypes = [_d, _d, _d, C.POINTER(_d)]
    L.uot_convergence_error.argtypes = [_P, _u64, _P, _u64]
    L.uot_convergence_error.restype = _d
    L.uot_rank_partition.argtypes = [_u64, _u64, _P]
    L.uot_gen_problem_f32.argtypes = [_u64, _u64, _u64, _P, _P, _P, _i]
    L.uot_gen_block_f32.argtypes = [_u64, _u64, _u64, _u64, _u64, _P, _P, _P, _i]
    L.uot_host_alloc.argtypes = [_u64]
    L.uot_host_alloc.restype = _P
    L.uot_host_free.argtypes = [_P]
    L.uot_host_free.restype = None
    _lib = L
    return L


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _raise(code: int, what: str):
    raise _ERRORS.get(code, Error)(what)


# ------------------------------------------------------------------ types --


@dataclass
class Problem:
    """Problem<float> (problem.hpp:19-28): a (M x N), rpd (M), cpd (N), er, ep."""
    a: np.ndarray
    rpd: np.ndarray
    cpd: np.ndarray
    er: float = 1.0
    ep: float = 1.0

    def m(self) -> int:
        return int(self.a.shape[0])

    def n(self) -> int:
        return int(self.a.shape[1])


@dataclass
class ScalingFactors:
    alpha: np.ndarray = field(default_factory=lambda: np.empty(0))
    beta: np.ndarray = field(default_factory=lambda: np.empty(0))


@dataclass
class SolveReport:
    solver: str = ""
    iterations: int = 0
    final_error: float = 0.0
    converged: bool = False
    wall_ms: float = 0.0


@dataclass
class SolveResult:
    plan: np.ndarray
    factors: ScalingFactors
    report: SolveReport


@dataclass
class FusedState:
    col_sums: np.ndarray


@dataclass
class CommStats:
    """CommStats (distributed.hpp:24-27)."""
    allreduce_calls: int = 0
    doubles_reduced: int = 0


@dataclass
class DistributedResult:
    """DistributedResult<T> (distributed.hpp:34-40). From distributed_solve (one
    process, every rank): the whole plan and alpha. From the per-process
    distributed.distributed_solve: THIS rank's rows [row_begin, row_end)."""
    plan: np.ndarray
    factors: "ScalingFactors"
    report: "SolveReport"
    comm: CommStats = field(default_factory=CommStats)
    row_begin: int = 0
    row_end: int = 0


@dataclass
class RankPartition:
    ranks: int
    blocks: list  # [(begin, end)]

    @staticmethod
    def make(ranks: int, rows: int) -> "RankPartition":
        b = np.zeros(max(int(ranks), 0) + 1, np.uint64)
        rc = lib().uot_rank_partition(int(ranks), int(rows), _ptr(b))
        if rc:
            _raise(rc, f"RankPartition: {ranks} ranks for {rows} rows would leave a rank without rows")
        return RankPartition(int(ranks), [(int(b[r]), int(b[r + 1])) for r in range(int(ranks))])


# ----------------------------------------------------------------- scalars --


def compute_fi(er: float, ep: float) -> float:
    out = _d()
    if lib().uot_compute_fi(float(er), float(ep), C.byref(out)):
        _raise(1, "compute_fi: er must be positive and finite, ep non-negative and finite")
    return out.value


def rescale_factor(target: float, s: float, fi: float) -> float:
    out = _d()
    if lib().uot_rescale_factor(float(target), float(s), float(fi), C.byref(out)):
        _raise(2, "rescale_factor: slice sum is not strictly positive or factor left the positive finite range")
    return out.value


def convergence_error(f: ScalingFactors) -> float:
    a = np.ascontiguousarray(f.alpha, np.float64)
    b = np.ascontiguousarray(f.beta, np.float64)
    return lib().uot_convergence_error(_ptr(a), a.size, _ptr(b), b.size)


class PinnedBuffer:
    """Page-locked host array (cudaMallocHost) exposed as a numpy array."""

    def __init__(self, shape, dtype):
        self.dtype = np.dtype(dtype)
        n = int(np.prod(shape)) * self.dtype.itemsize
        self._p = lib().uot_host_alloc(n)
        if not self._p:
            raise CudaError(f"cudaMallocHost({n}) failed")
        self.array = np.ctypeslib.as_array((C.c_uint8 * n).from_address(self._p)).view(self.dtype).reshape(shape)

    def free(self):
        if self._p:
            self.array = None
            lib().uot_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass


def gen_block(seed: int, global_rows: int, n: int, row0: int, rows: int, threads: int = 0,
              out: np.ndarray | None = None, dtype=np.float32) -> Problem:
    """Rows [row0, row0+rows) of gen_problem_t<T>(seed, global_rows, n) (T = float
    or double): the rank-local block of a row-sharded problem (A block, rpd
    slice, full cpd)."""
    dtype = np.dtype(dtype) if out is None else out.dtype
    a = np.empty((rows, n), dtype) if out is None else out
    rpd = np.empty(rows, np.float64)
    cpd = np.empty(n, np.float64)
    fn = lib().uot_gen_block_f64 if dtype == np.float64 else lib().uot_gen_block_f32
    rc = fn(int(seed), int(global_rows), int(n), int(row0), int(rows), _ptr(a), _ptr(rpd), _ptr(cpd),
            threads or (os.cpu_count() or 1))
    if rc:
        _raise(rc, "gen_block: bad block")
    return Problem(a, rpd, cpd, 1.0, 1.0)


def gen_problem_t(seed: int, m: int, n: int, threads: int = 0, out: np.ndarray | None = None,
                  dtype=np.float32) -> Problem:
    """gen_problem_t<T> (problem_io.hpp:17-31), T = float (default) or double;
    er = ep = 1. `out` may be a preallocated (m, n) array (e.g. PinnedBuffer.array)."""
    if m < 1 or n < 1:
        _raise(1, "gen_problem: matrix must be at least 1x1")
    return gen_block(seed, m, n, 0, m, threads, out, dtype)


# ---------------------------------------------------------- problem files --


def problem_file_info(path) -> dict:
    """The header of a .uotp file, with read_problem's checks (problem_io.cpp:106-135)."""
    m, n, dt, er, ep = _u64(), _u64(), _i(), _d(), _d()
    rc = lib().uot_problem_file_info(os.fsencode(path), C.byref(m), C.byref(n), C.byref(dt), C.byref(er),
                                     C.byref(ep))
    if rc:
        _raise(rc, lib().uot_last_io_error().decode())
    return {"m": int(m.value), "n": int(n.value), "dtype": {1: "f32", 2: "f64"}[dt.value],
            "er": float(er.value), "ep": float(ep.value)}


def read_problem(path) -> Problem:
    """read_problem (problem_io.cpp:106-141) on the host: a Problem<float> or
    Problem<double> (the matrix dtype says which)."""
    info = problem_file_info(path)
    m, n = info["m"], info["n"]
    es, code = (8, "<f8") if info["dtype"] == "f64" else (4, "<f4")
    raw = np.fromfile(path, dtype=np.uint8, offset=40)
    a = raw[: es * m * n].view(code).reshape(m, n)
    rpd = raw[es * m * n: es * m * n + 8 * m].view("<f8")
    cpd = raw[es * m * n + 8 * m:].view("<f8")
    dt = np.float64 if es == 8 else np.float32
    return Problem(a.astype(dt), rpd.astype(np.float64), cpd.astype(np.float64), info["er"], info["ep"])


def write_problem(path, p: Problem):
    """write_problem (problem_io.cpp:97-104) of a Problem<float> or Problem<double>."""
    f64 = np.asarray(p.a).dtype == np.float64
    a = np.ascontiguousarray(p.a, "<f8" if f64 else "<f4")
    hdr = bytearray(b"UOTP") + (1).to_bytes(2, "little") + (2 if f64 else 1).to_bytes(2, "little")
    hdr += int(a.shape[0]).to_bytes(8, "little") + int(a.shape[1]).to_bytes(8, "little")
    hdr += np.array([p.er, p.ep], "<f8").tobytes()
    with open(path, "wb") as f:
        f.write(bytes(hdr))
        f.write(a.tobytes())
        f.write(np.ascontiguousarray(p.rpd, "<f8").tobytes())
        f.write(np.ascontiguousarray(p.cpd, "<f8").tobytes())


# ---------------------------------------------------------------- session --


class Session:
    """A problem resident in HBM on one GPU (or one rank's row block of it).

    The device-resident form of fused_solve's loop (fused.hpp:259-285):
    set_problem -> init_col_sums -> iterate(k, tol) -> factors()/plan().
    """

    def __init__(self, rows: int, cols: int, device: int = 0, *, dist=None, dtype=np.float32):
        """dtype: np.float32 (Problem<float>) or np.float64 (Problem<double>)."""
        self._h = _P()
        L = lib()
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.float32, np.float64):
            _raise(1, f"dtype {self.dtype}: Problem<float> or Problem<double> only")
        code = UOT_F64 if self.dtype == np.float64 else UOT_F32
        if dist is None:
            rc = L.uot_create(C.byref(self._h), int(rows), int(cols), code, int(device))
        elif dist[2] == "peer":  # (rank, nranks, "peer"): connect() with every rank's handle next
            rank, nranks, _ = dist
            rc = L.uot_create_peer(C.byref(self._h), int(rows), int(cols), code, int(device),
                                   int(rank), int(nranks))
        else:
            rank, nranks, nccl_id = dist
            idp = None  # NULL: a one-rank session without a communicator
            if nccl_id is not None:
                idbuf = (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id).ljust(128, b"\0"))
                idp = C.cast(idbuf, _P)
            rc = L.uot_create_dist(C.byref(self._h), int(rows), int(cols), code, int(device),
                                   int(rank), int(nranks), idp)
        if rc:
            msg = self._err()
            self.close()
            _raise(rc, msg)
        lay = Layout()
        L.uot_get_layout(self._h, C.byref(lay))
        self.layout = lay.as_dict()
        self.rows = int(lay.rows)
        self.cols = int(lay.cols)
        self.row_offset = int(lay.row_offset)

    @classmethod
    def _adopt(cls, handle, dtype) -> "Session":
        """Wrap a session created elsewhere (uot_create_group)."""
        self = cls.__new__(cls)
        self._h = handle
        self.dtype = np.dtype(dtype)
        lay = Layout()
        lib().uot_get_layout(self._h, C.byref(lay))
        self.layout = lay.as_dict()
        self.rows, self.cols, self.row_offset = int(lay.rows), int(lay.cols), int(lay.row_offset)
        return self

    # -- plumbing
    def _err(self) -> str:
        return lib().uot_last_error(self._h).decode() if self._h else "session creation failed"

    def _check(self, rc: int):
        if rc:
            _raise(rc, self._err())

    def close(self):
        if self._h:
            lib().uot_destroy(self._h)
            self._h = _P()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @property
    def stream(self) -> int:
        return int(lib().uot_get_stream(self._h) or 0)

    # -- problem
    def set_problem(self, p: Problem):
        a = np.ascontiguousarray(p.a, self.dtype)
        if a.shape != (self.rows, self.cols):
            _raise(1, f"matrix shape {a.shape} does not match the session ({self.rows}, {self.cols})")
        rpd = np.ascontiguousarray(p.rpd, np.float64)
        cpd = np.ascontiguousarray(p.cpd, np.float64)
        if rpd.size != self.rows:
            _raise(1, f"row-marginal length {rpd.size} does not match row count {self.rows}")
        if cpd.size != self.cols:
            _raise(1, f"column-marginal length {cpd.size} does not match column count {self.cols}")
        fn = lib().uot_set_problem_f64 if self.dtype == np.float64 else lib().uot_set_problem
        self._check(fn(self._h, _ptr(a), _ptr(rpd), _ptr(cpd), float(p.er), float(p.ep)))

    def load_problem_file(self, path):
        """read_problem (problem_io.cpp:106-141) of this session's row block,
        streamed from the .uotp file straight to HBM, then validated."""
        self._check(lib().uot_load_problem_file(self._h, os.fsencode(path)))

    def save_problem_file(self, path):
        """write_problem (problem_io.cpp:97-104) of the current plan with the
        session's marginals and er/ep (collective over the ranks)."""
        self._check(lib().uot_save_problem_file(self._h, os.fsencode(path)))

    def set_iterate_input(self, a: np.ndarray, rpd: np.ndarray, cpd: np.ndarray, fi: float):
        """fused_iterate's inputs as given (uot_set_iterate_input): the current
        plan, marginals and fi, without require_valid's checks."""
        a = np.ascontiguousarray(a, self.dtype)
        if a.shape != (self.rows, self.cols):
            _raise(1, f"matrix shape {a.shape} does not match the session ({self.rows}, {self.cols})")
        rpd = np.ascontiguousarray(rpd, np.float64)
        cpd = np.ascontiguousarray(cpd, np.float64)
        if rpd.size != self.rows or cpd.size != self.cols:
            _raise(1, "marginal lengths do not match the matrix")
        code = UOT_F64 if self.dtype == np.float64 else UOT_F32
        self._check(lib().uot_set_iterate_input(self._h, _ptr(a), code, _ptr(rpd), _ptr(cpd), float(fi)))

    def set_fi(self, fi: float):
        self._check(lib().uot_set_fi(self._h, float(fi)))

    def generate_problem(self, seed: int, er: float = 1.0, ep: float = 1.0):
        self._check(lib().uot_generate_problem(self._h, int(seed), float(er), float(ep)))

    def set_plan(self, a: np.ndarray):
        a = np.ascontiguousarray(a, self.dtype)
        if a.shape != (self.rows, self.cols):
            _raise(1, "fused_iterate: matrix shape does not match problem")
        fn = lib().uot_set_plan_f64 if self.dtype == np.float64 else lib().uot_set_plan
        self._check(fn(self._h, _ptr(a)))

    # -- the path
    def init_col_sums(self):
        self._check(lib().uot_init_col_sums(self._h))

    def set_col_sums(self, cs: np.ndarray):
        cs = np.ascontiguousarray(cs, np.float64)
        if cs.size != self.cols:
            _raise(1, "fused_iterate: carried column sums have wrong length")
        self._check(lib().uot_set_col_sums(self._h, _ptr(cs)))

    def col_sums(self) -> np.ndarray:
        out = np.empty(self.cols, np.float64)
        self._check(lib().uot_get_col_sums(self._h, _ptr(out)))
        return out

    def iterate(self, k: int = 1, tol: float = 1e-300):
        """Up to k iterations; returns (iterations, final_error, converged)."""
        it, err, conv = _u64(), _d(), _i()
        self._check(lib().uot_iterate(self._h, int(k), float(tol), C.byref(it), C.byref(err), C.byref(conv)))
        return int(it.value), float(err.value), bool(conv.value)

    def iterate_timed(self, k: int = 1, tol: float = 1e-300):
        """iterate() plus the device milliseconds of the k iterations (CUDA events)."""
        it, err, conv, ms = _u64(), _d(), _i(), _d()
        self._check(lib().uot_iterate_timed(self._h, int(k), float(tol), C.byref(it), C.byref(err),
                                            C.byref(conv), C.byref(ms)))
        return int(it.value), float(err.value), bool(conv.value), float(ms.value)

    def synchronize(self):
        self._check(lib().uot_synchronize(self._h))

    def factors(self) -> ScalingFactors:
        alpha = np.empty(self.rows, np.float64)
        beta = np.empty(self.cols, np.float64)
        self._check(lib().uot_get_factors(self._h, _ptr(alpha), _ptr(beta)))
        return ScalingFactors(alpha, beta)

    def plan(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.rows, self.cols), self.dtype)
        if out.dtype != self.dtype or out.shape != (self.rows, self.cols) or not out.flags.c_contiguous:
            _raise(1, f"plan buffer must be a C-contiguous {self.dtype} array of shape ({self.rows}, {self.cols})")
        fn = lib().uot_get_plan_f64 if self.dtype == np.float64 else lib().uot_get_plan
        self._check(fn(self._h, _ptr(out)))
        return out

    def report(self):
        it, err, conv = _u64(), _d(), _i()
        self._check(lib().uot_get_report(self._h, C.byref(it), C.byref(err), C.byref(conv)))
        return int(it.value), float(err.value), bool(conv.value)

    def comm_stats(self):
        calls, dbl = _u64(), _u64()
        self._check(lib().uot_get_comm_stats(self._h, C.byref(calls), C.byref(dbl)))
        return int(calls.value), int(dbl.value)

    VARIANTS = {"fused": 0, "two_pass": 1, "baseline": 2}

    def set_variant(self, name: str):
        """Iteration schedule: "fused" (the product), or the ablations "two_pass"
        (tiled.hpp:210-229) and "baseline" (baseline.hpp:100-110)."""
        if name not in self.VARIANTS:
            _raise(1, f"unknown iteration variant {name!r}")
        self._check(lib().uot_set_variant(self._h, self.VARIANTS[name]))

    SCHEDULES = {"uniform": 0, "weighted": 1, "dynamic": 2}

    def set_schedule(self, name: str):
        """Row-batch schedule of the sweep (uot_set_schedule): "uniform"
        (default; balanced_blocks, bit-reproducible), "weighted" (static blocks
        from group weights, bit-reproducible for given weights) or "dynamic"."""
        if name not in self.SCHEDULES:
            _raise(1, f"unknown schedule {name!r}")
        self._check(lib().uot_set_schedule(self._h, self.SCHEDULES[name]))
        self._refresh_layout()

    def set_group_weights(self, w):
        """Per-row-group weights (uot_set_group_weights); selects "weighted"."""
        w = np.ascontiguousarray(w, np.uint32)
        self._check(lib().uot_set_group_weights(self._h, _ptr(w), w.size))
        self._refresh_layout()

    def group_weights(self) -> np.ndarray:
        w = np.zeros(self.layout["groups"], np.uint32)
        self._check(lib().uot_get_group_weights(self._h, _ptr(w), w.size))
        return w

    def calibrate_schedule(self, k: int = 4) -> np.ndarray:
        """Measure per-group weights with k dynamic iterations on a scratch copy
        of the plan (uot_calibrate_schedule); selects "weighted"."""
        self._check(lib().uot_calibrate_schedule(self._h, int(k)))
        self._refresh_layout()
        return self.group_weights()

    def set_deterministic(self, on: bool = True):
        """on: a static schedule (weighted when weights are set, else uniform;
        bit-reproducible run to run); off: the dynamic batch counter."""
        self._check(lib().uot_set_deterministic(self._h, 1 if on else 0))
        self._refresh_layout()

    def _refresh_layout(self):
        lay = Layout()
        lib().uot_get_layout(self._h, C.byref(lay))
        self.layout = lay.as_dict()

    def schedule_stats(self):
        """Per CTA slot: SM id and row batches of the last sweep; per group: class weight (1/32)."""
        grid = self.layout["groups"] * self.layout["G"]
        smid = np.zeros(grid, np.uint32)
        nb = np.zeros(grid, np.uint32)
        w = np.zeros(self.layout["groups"], np.uint32)
        self._check(lib().uot_get_schedule_stats(self._h, _ptr(smid), _ptr(nb), _ptr(w)))
        return smid, nb, w

    def set_resident(self, on: bool = True):
        """Allow (default) or forbid the one-launch resident solve for small
        problems (uot_set_resident)."""
        self._check(lib().uot_set_resident(self._h, 1 if on else 0))
        self._refresh_layout()

    def set_timing(self, on: bool = True):
        self._check(lib().uot_set_timing(self._h, 1 if on else 0))

    def timing(self):
        s, f, n = _d(), _d(), _u64()
        self._check(lib().uot_get_timing(self._h, C.byref(s), C.byref(f), C.byref(n)))
        return float(s.value), float(f.value), int(n.value)

    def kernel_launches(self) -> int:
        return int(lib().uot_kernel_launches(self._h))


# ------------------------------------------------------------- solver API --


class SessionGroup:
    """Every rank of a row-sharded problem in THIS process (uot_create_group):
    rank r is a Session over its RankPartition block on devices[r] (default:
    round robin over the visible GPUs; ranks may share one), exchange regions
    mapped directly between the ranks. init_col_sums / iterate are collective
    over the ranks (uot_group_*); everything else is per rank (`ranks[r]`)."""

    def __init__(self, global_rows: int, cols: int, nranks: int, devices=None, partition=None,
                 dtype=np.float32):
        L = lib()
        self.dtype = np.dtype(dtype)
        code = UOT_F64 if self.dtype == np.float64 else UOT_F32
        n = int(nranks)
        hs = (_P * max(n, 1))()
        dev = None if devices is None else np.ascontiguousarray(devices, np.int32)
        if dev is not None and dev.shape != (n,):
            _raise(1, f"SessionGroup: {dev.size} devices for {n} ranks")
        bnd = None
        if partition is not None:
            if partition.ranks != n or len(partition.blocks) != n:
                _raise(3, "distributed_solve: partition does not cover the matrix rows")
            bnd = np.array([0] + [e for _, e in partition.blocks], np.uint64)
            if any(b != bnd[i] for i, (b, _) in enumerate(partition.blocks)):
                _raise(3, "distributed_solve: partition blocks are not contiguous")
        rc = L.uot_create_group(C.cast(hs, _P), int(global_rows), int(cols), code, _ptr(dev), n, _ptr(bnd))
        self.ranks = []
        for r in range(n):
            if hs[r]:
                self.ranks.append(Session._adopt(_P(hs[r]), self.dtype))
        if rc:
            msg = next((x._err() for x in reversed(self.ranks)), "session group creation failed")
            self.close()
            _raise(rc, msg)
        self._hs = hs

    def _check(self, rc: int):
        if rc:
            msg = "; ".join(f"rank {r}: {x._err()}" for r, x in enumerate(self.ranks) if x._err())
            _raise(rc, msg or "session group call failed")

    def init_col_sums(self):
        self._check(lib().uot_group_init_col_sums(C.cast(self._hs, _P), len(self.ranks)))

    def iterate(self, k: int = 1, tol: float = 1e-300):
        it, err, conv = _u64(), _d(), _i()
        self._check(lib().uot_group_iterate(C.cast(self._hs, _P), len(self.ranks), int(k), float(tol),
                                            C.byref(it), C.byref(err), C.byref(conv)))
        return int(it.value), float(err.value), bool(conv.value)

    def close(self):
        for x in self.ranks:
            x.close()
        self.ranks = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def distributed_solve(p: Problem, tol: float, max_iter: int, ranks=1, devices=None) -> DistributedResult:
    """distributed_solve(p, tol, max_iter, ranks | RankPartition) (distributed.hpp:52-142)
    in one process: every rank on a GPU (devices[r], default round robin), one
    fused peer-memory exchange of the column sums per iteration, the whole plan
    and alpha assembled on the host as in the reference."""
    _validate_controls(tol, max_iter, "distributed_solve")
    t0 = time.perf_counter()
    part = ranks if isinstance(ranks, RankPartition) else RankPartition.make(int(ranks), p.m())
    dt = np.float64 if np.asarray(p.a).dtype == np.float64 else np.float32
    plan = np.empty((p.m(), p.n()), dt)
    alpha = np.empty(p.m())
    with SessionGroup(p.m(), p.n(), part.ranks, devices, part, dt) as g:
        for s in g.ranks:
            b, e = s.row_offset, s.row_offset + s.rows
            s.set_problem(Problem(p.a[b:e], p.rpd[b:e], p.cpd, p.er, p.ep))
        g.init_col_sums()
        it, err, conv = g.iterate(max_iter, tol)
        for s in g.ranks:
            b, e = s.row_offset, s.row_offset + s.rows
            f = s.factors()
            alpha[b:e] = f.alpha
            s.plan(out=plan[b:e])
        beta = f.beta
    rep = SolveReport("dist", it, err, conv, (time.perf_counter() - t0) * 1e3)
    return DistributedResult(plan, ScalingFactors(alpha, beta), rep, CommStats(it, it * p.n()), 0, p.m())


def _validate_controls(tol: float, max_iter: int, who: str):
    if not (tol > 0.0):
        _raise(1, f"{who}: tol must be positive")
    if max_iter < 1:
        _raise(1, f"{who}: max_iter must be at least 1")


def fused_solve(p: Problem, tol: float, max_iter: int, device: int = 0,
                session: Session | None = None) -> SolveResult:
    """fused_solve (fused.hpp:259-285) on one B200.

    report.wall_ms covers upload, seed, iterations and download (the reference's
    covers seed + iterations of an in-memory matrix)."""
    _validate_controls(tol, max_iter, "fused_solve")
    t0 = time.perf_counter()
    own = session is None
    dt = np.float64 if np.asarray(p.a).dtype == np.float64 else np.float32  # Problem<double> stays double
    s = Session(p.m(), p.n(), device, dtype=dt) if own else session
    try:
        s.set_problem(p)
        s.init_col_sums()
        it, err, conv = s.iterate(max_iter, tol)
        f = s.factors()
        plan = s.plan()
    finally:
        if own:
            s.close()
    rep = SolveReport("cuda", it, err, conv, (time.perf_counter() - t0) * 1e3)
    return SolveResult(plan, f, rep)


def init_col_sums(a: np.ndarray, device: int = 0) -> np.ndarray:
    """init_col_sums (fused.hpp:71-110) of a host matrix, computed on the GPU."""
    a = np.ascontiguousarray(a, np.float32)
    m, n = a.shape
    with Session(m, n, device) as s:
        s.set_problem(Problem(a, np.ones(m), np.ones(n), 1.0, 1.0))
        s.init_col_sums()
        return s.col_sums()


def fused_iterate(a: np.ndarray, state: FusedState, p: Problem, fi: float, device: int = 0,
                  session: Session | None = None) -> ScalingFactors:
    """fused_iterate (fused.hpp:164-191) with the reference's host-in/host-out
    contract: `a` and `state.col_sums` are updated in place. Matrix<float> or
    Matrix<double> by a's dtype (Problem<double> iterates in f64, as the
    reference's template does). Like the reference it checks only shapes: the
    current plan and fi are used as given (no require_valid). Each call moves
    the matrix over PCIe; keep a Session for device-resident loops."""
    if a.shape != (p.m(), p.n()):
        _raise(1, "fused_iterate: matrix shape does not match problem")
    if np.asarray(state.col_sums).size != p.n():
        _raise(1, "fused_iterate: carried column sums have wrong length")
    dt = np.dtype(np.float64 if a.dtype == np.float64 else np.float32)
    s = session if session is not None else _cached_session(p.m(), p.n(), device, dt)
    if s.dtype != dt:
        _raise(1, f"fused_iterate: a {a.dtype} matrix on a {s.dtype} session")
    s.set_iterate_input(a, p.rpd, p.cpd, fi)
    s.set_col_sums(state.col_sums)
    s.iterate(1, 1e-300)
    f = s.factors()
    s.plan(out=a) if a.flags.c_contiguous and a.dtype == dt else a.__setitem__(Ellipsis, s.plan())
    state.col_sums = s.col_sums()
    return f


_tls = threading.local()


def _cached_session(m: int, n: int, device: int, dtype=np.float32) -> "Session":
    """One session per thread and (shape, device, dtype), kept between
    fused_iterate calls: a loop pays the two PCIe transfers per call, not a
    session setup."""
    key = (int(m), int(n), int(device), np.dtype(dtype).str)
    s = getattr(_tls, "session", None)
    if s is None or getattr(_tls, "key", None) != key or not s._h:
        if s is not None:
            s.close()
        _tls.session, _tls.key = Session(m, n, device, dtype=dtype), key
    return _tls.session

