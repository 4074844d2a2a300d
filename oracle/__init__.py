"""CPU oracle for the fused Sinkhorn-UOT path — TEST INFRASTRUCTURE ONLY.

Two checkers behind one numpy interface:

* ``Oracle()``    — the plain-C restatement (oracle/uot_oracle.c -> liboracle.so);
* ``RefOracle()`` — the UNMODIFIED reference compiled from /root/reference by
  oracle/Makefile (-> oracle/_ref/libuot_ref.so). Present wherever the built
  .so travelled; building it needs /root/reference (this container only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. The product
(paper_2412_11079_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libuot_ref.so")
REF_TREE = "/root/reference/proj/core"

_u64, _sz, _d, _i = C.c_uint64, C.c_size_t, C.c_double, C.c_int
_pf = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_pd = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_P = C.c_void_p

STATUS_NAMES = {0: "ok", 1: "InvalidParameter", 2: "DegenerateSum", 3: "PartitionError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {what}")
        self.code = code


def build(ref: bool = False) -> None:
    """Compile liboracle.so (and _ref when the reference tree is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir(REF_TREE):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


@dataclass
class SolveOut:
    plan: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray
    iterations: int
    final_error: float
    converged: bool
    col_sums: np.ndarray | None = None
    allreduce_calls: int = 0
    doubles_reduced: int = 0


class Oracle:
    """ctypes front of oracle/uot_oracle.c (see that file for the citations)."""

    def __init__(self):
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(
            os.path.join(HERE, "uot_oracle.c")
        ):
            build()
        self.lib = C.CDLL(LIB)
        L = self.lib
        L.orc_splitmix64_next.argtypes = [C.POINTER(_u64)]
        L.orc_splitmix64_next.restype = _u64
        L.orc_next_unit.argtypes = [C.POINTER(_u64)]
        L.orc_next_unit.restype = _d
        L.orc_gen_problem_f32.argtypes = [_u64, _sz, _sz, _P, _P, _P, _i]
        L.orc_gen_problem_f64.argtypes = [_u64, _sz, _sz, _P, _P, _P, _i]
        L.orc_compute_fi.argtypes = [_d, _d, C.POINTER(_d)]
        L.orc_rescale_factor.argtypes = [_d, _d, _d, C.POINTER(_d)]
        L.orc_convergence_error.argtypes = [_P, _sz, _P, _sz]
        L.orc_convergence_error.restype = _d
        L.orc_balanced_blocks.argtypes = [_sz, _sz, _P]
        L.orc_rank_partition.argtypes = [_sz, _sz, _P]
        L.orc_init_col_sums_f32.argtypes = [_P, _sz, _sz, _sz, _P]
        L.orc_beta_from_state.argtypes = [_P, _P, _sz, _d, _P]
        L.orc_fused_row_pass_f32.argtypes = [_P, _sz, _P, _d, _d, _P, C.POINTER(_d)]
        L.orc_fused_iterate_f32.argtypes = [_P, _sz, _sz, _P, _P, _P, _d, _sz, _P, _P]
        solve_args = [_P, _sz, _sz, _P, _P, _d, _d, _d, _sz, _sz, _P, _P, _P,
                      C.POINTER(_sz), C.POINTER(_d), C.POINTER(_i)]
        L.orc_fused_solve_f32.argtypes = solve_args
        L.orc_fused_solve_f64.argtypes = solve_args
        L.orc_distributed_solve_f32.argtypes = [
            _P, _sz, _sz, _P, _P, _d, _d, _d, _sz, _sz, _P, _P,
            C.POINTER(_sz), C.POINTER(_d), C.POINTER(_i), C.POINTER(_u64), C.POINTER(_u64)]
        L.orc_allreduce_vectors.argtypes = [_P, _sz, _sz, _P]

    @staticmethod
    def _check(code):
        if code != 0:
            raise OracleError(code)

    # -- inputs (problem_io.hpp:17-31) ------------------------------------
    def gen_problem(self, seed: int, m: int, n: int, dtype=np.float32, threads: int = 0):
        threads = threads or (os.cpu_count() or 1)
        a = np.empty((m, n), dtype=dtype)
        rpd = np.empty(m, np.float64)
        cpd = np.empty(n, np.float64)
        fn = self.lib.orc_gen_problem_f32 if dtype == np.float32 else self.lib.orc_gen_problem_f64
        self._check(fn(seed, m, n, _ptr(a), _ptr(rpd), _ptr(cpd), threads))
        return a, rpd, cpd

    # -- scalars (scaling.cpp:9-29) -----------------------------------------
    def compute_fi(self, er, ep):
        out = _d()
        self._check(self.lib.orc_compute_fi(er, ep, C.byref(out)))
        return out.value

    def rescale_factor(self, t, s, fi):
        out = _d()
        self._check(self.lib.orc_rescale_factor(t, s, fi, C.byref(out)))
        return out.value

    def convergence_error(self, alpha, beta):
        alpha = np.ascontiguousarray(alpha, np.float64)
        beta = np.ascontiguousarray(beta, np.float64)
        return self.lib.orc_convergence_error(_ptr(alpha), alpha.size, _ptr(beta), beta.size)

    def balanced_blocks(self, k, rows):
        b = np.empty(k + 1, np.uint64)
        self.lib.orc_balanced_blocks(k, rows, _ptr(b))
        return [int(x) for x in b]

    def rank_partition(self, ranks, rows):
        b = np.zeros(max(ranks, 0) + 1, np.uint64)
        self._check(self.lib.orc_rank_partition(ranks, rows, _ptr(b)))
        return [int(x) for x in b]

    # -- the path -----------------------------------------------------------
    def init_col_sums(self, a, nblocks=1):
        a = np.ascontiguousarray(a, np.float32)
        cs = np.empty(a.shape[1], np.float64)
        self.lib.orc_init_col_sums_f32(_ptr(a), a.shape[0], a.shape[1], nblocks, _ptr(cs))
        return cs

    def fused_iterate(self, a, col_sums, rpd, cpd, fi, workers=1):
        """One fused_iterate_parallel; a and col_sums are updated in place."""
        m, n = a.shape
        alpha = np.empty(m, np.float64)
        beta = np.empty(n, np.float64)
        self._check(self.lib.orc_fused_iterate_f32(_ptr(a), m, n, _ptr(col_sums), _ptr(rpd),
                                                   _ptr(cpd), fi, workers, _ptr(alpha), _ptr(beta)))
        return alpha, beta

    def fused_solve(self, a, rpd, cpd, er, ep, tol, max_iter, workers=1) -> SolveOut:
        plan = np.array(a, copy=True, order="C")
        m, n = plan.shape
        alpha = np.empty(m, np.float64)
        beta = np.empty(n, np.float64)
        cs = np.empty(n, np.float64)
        it, err, conv = _sz(), _d(), _i()
        fn = self.lib.orc_fused_solve_f32 if plan.dtype == np.float32 else self.lib.orc_fused_solve_f64
        self._check(fn(_ptr(plan), m, n, _ptr(rpd), _ptr(cpd), er, ep, tol, max_iter, workers,
                       _ptr(alpha), _ptr(beta), _ptr(cs), C.byref(it), C.byref(err), C.byref(conv)))
        return SolveOut(plan, alpha, beta, it.value, err.value, bool(conv.value), cs)

    def distributed_solve(self, a, rpd, cpd, er, ep, tol, max_iter, ranks) -> SolveOut:
        plan = np.array(a, dtype=np.float32, copy=True, order="C")
        m, n = plan.shape
        alpha = np.empty(m, np.float64)
        beta = np.empty(n, np.float64)
        it, err, conv, calls, dbl = _sz(), _d(), _i(), _u64(), _u64()
        self._check(self.lib.orc_distributed_solve_f32(
            _ptr(plan), m, n, _ptr(rpd), _ptr(cpd), er, ep, tol, max_iter, ranks, _ptr(alpha),
            _ptr(beta), C.byref(it), C.byref(err), C.byref(conv), C.byref(calls), C.byref(dbl)))
        return SolveOut(plan, alpha, beta, it.value, err.value, bool(conv.value), None,
                        calls.value, dbl.value)


class RefOracle:
    """The reference itself (oracle/_ref/libuot_ref.so, see oracle/ref_shim.cpp)."""

    def __init__(self):
        if not os.path.exists(REF_LIB):
            if os.path.isdir(REF_TREE):
                build(ref=True)
            else:
                raise FileNotFoundError(
                    "oracle/_ref/libuot_ref.so missing and /root/reference is absent here")
        self.lib = C.CDLL(REF_LIB)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_gen_problem_f32.argtypes = [_u64, _sz, _sz, _P, _P, _P]
        solve = [_P, _sz, _sz, _P, _P, _d, _d, _d, _sz, _sz, _P, _P, _P,
                 C.POINTER(_sz), C.POINTER(_d), C.POINTER(_i)]
        L.ref_fused_solve_f32.argtypes = solve
        L.ref_fused_solve_f64.argtypes = solve
        L.ref_fused_iterate_k_f32.argtypes = [_P, _sz, _sz, _P, _P, _d, _d, _sz, _sz, _P, _P, _P,
                                              _P, C.POINTER(_d)]
        L.ref_time_fused_iterate_f32.argtypes = [_P, _sz, _sz, _P, _P, _d, _d, _sz, _sz, _P]
        L.ref_fused_iterate_k_inplace_f32.argtypes = [_P, _sz, _sz, _P, _P, _d, _d, _sz, _sz, _P, _P, _P,
                                                      C.POINTER(_d)]
        L.ref_distributed_solve_f32.argtypes = [
            _P, _sz, _sz, _P, _P, _d, _d, _d, _sz, _sz, _P, _P, _P,
            C.POINTER(_sz), C.POINTER(_d), C.POINTER(_i), C.POINTER(_u64), C.POINTER(_u64)]
        L.ref_baseline_solve_f32.argtypes = [_P, _sz, _sz, _P, _P, _d, _d, _d, _sz, _P, _P, _P,
                                             C.POINTER(_sz), C.POINTER(_d), C.POINTER(_i)]
        L.ref_compute_fi.argtypes = [_d, _d, C.POINTER(_d)]
        L.ref_rescale_factor.argtypes = [_d, _d, _d, C.POINTER(_d)]
        L.ref_rank_partition.argtypes = [_sz, _sz, _P]
        L.ref_write_problem_f32.argtypes = [C.c_char_p, _P, _sz, _sz, _P, _P, _d, _d]
        L.ref_write_problem_f64.argtypes = [C.c_char_p, _P, _sz, _sz, _P, _P, _d, _d]
        L.ref_read_problem_f32.argtypes = [C.c_char_p, C.POINTER(_sz), C.POINTER(_sz), C.POINTER(_i),
                                           C.POINTER(_d), C.POINTER(_d), _P, _P, _P]

    def _check(self, code):
        if code != 0:
            raise OracleError(code, self.lib.ref_last_error().decode())

    def gen_problem(self, seed, m, n):
        a = np.empty((m, n), np.float32)
        rpd = np.empty(m, np.float64)
        cpd = np.empty(n, np.float64)
        self._check(self.lib.ref_gen_problem_f32(seed, m, n, _ptr(a), _ptr(rpd), _ptr(cpd)))
        return a, rpd, cpd

    def compute_fi(self, er, ep):
        out = _d()
        self._check(self.lib.ref_compute_fi(er, ep, C.byref(out)))
        return out.value

    def rescale_factor(self, t, s, fi):
        out = _d()
        self._check(self.lib.ref_rescale_factor(t, s, fi, C.byref(out)))
        return out.value

    def rank_partition(self, ranks, rows):
        b = np.zeros(max(ranks, 0) + 1, np.uint64)
        self._check(self.lib.ref_rank_partition(ranks, rows, _ptr(b)))
        return [int(x) for x in b]

    def write_problem(self, path, a, rpd, cpd, er, ep):
        """uot::write_problem (problem_io.cpp:97-104), f32 or f64 by the dtype of `a`."""
        a = np.ascontiguousarray(a)
        fn = self.lib.ref_write_problem_f32 if a.dtype == np.float32 else self.lib.ref_write_problem_f64
        self._check(fn(os.fsencode(path), _ptr(a), a.shape[0], a.shape[1], _ptr(np.ascontiguousarray(rpd, np.float64)),
                       _ptr(np.ascontiguousarray(cpd, np.float64)), er, ep))

    def read_problem(self, path):
        """uot::read_problem (problem_io.cpp:106-141): (dtype, er, ep, a, rpd, cpd); f64 payload not returned."""
        m, n, dt, er, ep = _sz(), _sz(), _i(), _d(), _d()
        self._check(self.lib.ref_read_problem_f32(os.fsencode(path), C.byref(m), C.byref(n), C.byref(dt),
                                                  C.byref(er), C.byref(ep), None, None, None))
        if dt.value != 1:
            return "f64", er.value, ep.value, None, None, None
        a = np.empty((m.value, n.value), np.float32)
        rpd = np.empty(m.value, np.float64)
        cpd = np.empty(n.value, np.float64)
        self._check(self.lib.ref_read_problem_f32(os.fsencode(path), C.byref(m), C.byref(n), C.byref(dt),
                                                  C.byref(er), C.byref(ep), _ptr(a), _ptr(rpd), _ptr(cpd)))
        return "f32", er.value, ep.value, a, rpd, cpd

    def fused_solve(self, a, rpd, cpd, er, ep, tol, max_iter, workers=1) -> SolveOut:
        a = np.ascontiguousarray(a)
        m, n = a.shape
        plan = np.empty_like(a)
        alpha = np.empty(m, np.float64)
        beta = np.empty(n, np.float64)
        it, err, conv = _sz(), _d(), _i()
        fn = self.lib.ref_fused_solve_f32 if a.dtype == np.float32 else self.lib.ref_fused_solve_f64
        self._check(fn(_ptr(a), m, n, _ptr(rpd), _ptr(cpd), er, ep, tol, max_iter, workers,
                       _ptr(plan), _ptr(alpha), _ptr(beta), C.byref(it), C.byref(err),
                       C.byref(conv)))
        return SolveOut(plan, alpha, beta, it.value, err.value, bool(conv.value))

    def fused_iterate_k(self, a, rpd, cpd, er, ep, workers, k) -> SolveOut:
        a = np.ascontiguousarray(a, np.float32)
        m, n = a.shape
        plan = np.empty_like(a)
        alpha = np.empty(m, np.float64)
        beta = np.empty(n, np.float64)
        cs = np.empty(n, np.float64)
        err = _d()
        self._check(self.lib.ref_fused_iterate_k_f32(_ptr(a), m, n, _ptr(rpd), _ptr(cpd), er, ep,
                                                     workers, k, _ptr(plan), _ptr(alpha),
                                                     _ptr(beta), _ptr(cs), C.byref(err)))
        return SolveOut(plan, alpha, beta, k, err.value, False, cs)

    def fused_iterate_k_inplace(self, a, rpd, cpd, er, ep, workers, k) -> SolveOut:
        """fused_iterate_k with `a` (C-contiguous float32) overwritten by the
        plan: two host copies of the matrix instead of four (config 5)."""
        if a.dtype != np.float32 or not a.flags.c_contiguous:
            raise ValueError("a must be a C-contiguous float32 array")
        m, n = a.shape
        alpha = np.empty(m, np.float64)
        beta = np.empty(n, np.float64)
        cs = np.empty(n, np.float64)
        err = _d()
        self._check(self.lib.ref_fused_iterate_k_inplace_f32(_ptr(a), m, n, _ptr(rpd), _ptr(cpd), er, ep,
                                                             workers, k, _ptr(alpha), _ptr(beta), _ptr(cs),
                                                             C.byref(err)))
        return SolveOut(a, alpha, beta, k, err.value, False, cs)

    def time_fused_iterate(self, a, rpd, cpd, er, ep, workers, k):
        a = np.ascontiguousarray(a, np.float32)
        m, n = a.shape
        ms = np.empty(k, np.float64)
        self._check(self.lib.ref_time_fused_iterate_f32(_ptr(a), m, n, _ptr(rpd), _ptr(cpd), er,
                                                        ep, workers, k, _ptr(ms)))
        return ms

    def distributed_solve(self, a, rpd, cpd, er, ep, tol, max_iter, ranks) -> SolveOut:
        a = np.ascontiguousarray(a, np.float32)
        m, n = a.shape
        plan = np.empty_like(a)
        alpha = np.empty(m, np.float64)
        beta = np.empty(n, np.float64)
        it, err, conv, calls, dbl = _sz(), _d(), _i(), _u64(), _u64()
        self._check(self.lib.ref_distributed_solve_f32(
            _ptr(a), m, n, _ptr(rpd), _ptr(cpd), er, ep, tol, max_iter, ranks, _ptr(plan),
            _ptr(alpha), _ptr(beta), C.byref(it), C.byref(err), C.byref(conv), C.byref(calls),
            C.byref(dbl)))
        return SolveOut(plan, alpha, beta, it.value, err.value, bool(conv.value), None,
                        calls.value, dbl.value)

    def baseline_solve(self, a, rpd, cpd, er, ep, tol, max_iter) -> SolveOut:
        a = np.ascontiguousarray(a, np.float32)
        m, n = a.shape
        plan = np.empty_like(a)
        alpha = np.empty(m, np.float64)
        beta = np.empty(n, np.float64)
        it, err, conv = _sz(), _d(), _i()
        self._check(self.lib.ref_baseline_solve_f32(
            _ptr(a), m, n, _ptr(rpd), _ptr(cpd), er, ep, tol, max_iter, _ptr(plan), _ptr(alpha),
            _ptr(beta), C.byref(it), C.byref(err), C.byref(conv)))
        return SolveOut(plan, alpha, beta, it.value, err.value, bool(conv.value))


def have_ref() -> bool:
    return os.path.exists(REF_LIB) or os.path.isdir(REF_TREE)
