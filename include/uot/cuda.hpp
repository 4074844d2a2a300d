// uot/cuda.hpp — drop-in B200 backend for the reference solver API.
//
// Header-only C++ facade over the C ABI (include/uot_cuda.h). It is written
// against the reference's own types and exceptions
// (/root/reference/proj/core/include/uot: Problem<T>, Matrix<T>, FusedState,
// ScalingFactors, SolveResult<T>, DistributedResult<T>, InvalidParameter,
// DegenerateSum, PartitionError, ConfigError), so a reference user switches a
// call site by changing the namespace:
//
//   uot::fused_solve(p, tol, max_iter, workers)   ->  uot::cuda::fused_solve(p, tol, max_iter)
//   uot::fused_iterate(a, state, p, fi)           ->  uot::cuda::fused_iterate(a, state, p, fi)
//   uot::distributed_solve(p, tol, max_iter, P)   ->  uot::cuda::distributed_solve(p, tol, max_iter, rank, P, nccl_id)
//
// plus uot::cuda::Session for loops that should keep the matrix resident in HBM
// (the reference's per-iteration API moves the whole matrix every call).
// Include the reference headers first (uot/problem.hpp, uot/fused.hpp,
// uot/distributed.hpp) and link libuot_cuda.so. See INTEGRATION.md.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "uot/distributed.hpp"
#include "uot/error.hpp"
#include "uot/fused.hpp"
#include "uot/problem.hpp"
#include "uot_cuda.h"

namespace uot::cuda {

// Status code -> the reference exception hierarchy (error.hpp:9-37).
[[noreturn]] inline void raise(int code, const std::string& what) {
  switch (code) {
    case UOT_INVALID_PARAMETER: throw InvalidParameter(what);
    case UOT_DEGENERATE_SUM: throw DegenerateSum(what);
    case UOT_PARTITION_ERROR: throw PartitionError(what);
    case UOT_CONFIG_ERROR: throw ConfigError(what);
    default: throw Error("cuda backend: " + what);
  }
}

// A problem resident on one B200 (or one rank's row block of it).
class Session {
 public:
  Session(std::size_t rows, std::size_t cols, int device = 0) {
    check(uot_create(&ctx_, rows, cols, UOT_F32, device));
  }
  // Rank `rank` of `nranks`, rows split by RankPartition::make (plan.cpp:35-44).
  Session(std::size_t global_rows, std::size_t cols, int device, int rank, int nranks,
          const std::uint8_t* nccl_id) {
    check(uot_create_dist(&ctx_, global_rows, cols, UOT_F32, device, rank, nranks, nccl_id));
  }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;
  Session(Session&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}
  ~Session() { uot_destroy(ctx_); }

  uot_layout layout() const {
    uot_layout l{};
    check(uot_get_layout(ctx_, &l));
    return l;
  }
  std::size_t rows() const { return layout().rows; }
  std::size_t cols() const { return layout().cols; }

  // Problem<float> (problem.hpp:19-28); this rank's rows when distributed.
  void set_problem(const Problem<float>& p) {
    check(uot_set_problem(ctx_, p.a.data().data(), p.rpd.data(), p.cpd.data(), p.er, p.ep));
  }
  void set_fi(double fi) { check(uot_set_fi(ctx_, fi)); }
  void set_plan(const Matrix<float>& a) { check(uot_set_plan(ctx_, a.data().data())); }
  void init_col_sums() { check(uot_init_col_sums(ctx_)); }
  void set_state(const FusedState& st) { check(uot_set_col_sums(ctx_, st.col_sums.data())); }
  FusedState state() const {
    FusedState st{std::vector<double>(cols())};
    check(uot_get_col_sums(ctx_, st.col_sums.data()));
    return st;
  }

  struct Progress {
    std::size_t iterations = 0;
    double final_error = 0.0;
    bool converged = false;
  };
  // Up to k fused iterations on the device, stopping like fused_solve (fused.hpp:273-281).
  Progress iterate(std::size_t k, double tol = 1e-300) {
    std::uint64_t it = 0;
    double err = 0.0;
    int conv = 0;
    check(uot_iterate(ctx_, k, tol, &it, &err, &conv));
    return {static_cast<std::size_t>(it), err, conv != 0};
  }
  ScalingFactors factors() const {
    ScalingFactors f;
    f.alpha.resize(rows());
    f.beta.resize(cols());
    check(uot_get_factors(ctx_, f.alpha.data(), f.beta.data()));
    return f;
  }
  Matrix<float> plan() const {
    Matrix<float> m(rows(), cols());
    check(uot_get_plan(ctx_, m.data().data()));
    return m;
  }
  CommStats comm() const {
    CommStats c;
    std::uint64_t calls = 0, dbl = 0;
    check(uot_get_comm_stats(ctx_, &calls, &dbl));
    c.allreduce_calls = calls;
    c.doubles_reduced = dbl;
    return c;
  }

 private:
  void check(int rc) const {
    if (rc != UOT_OK) raise(rc, uot_last_error(ctx_));
  }
  uot_ctx* ctx_ = nullptr;
};

// fused_solve (fused.hpp:259-285) on one B200. The plan, factors and report
// have the reference's meaning; report.solver is "cuda" and wall_ms also
// covers the PCIe transfers.
inline SolveResult<float> fused_solve(const Problem<float>& p, double tol, std::size_t max_iter,
                                      int device = 0) {
  require_valid(p);
  if (!(tol > 0.0)) throw InvalidParameter("fused_solve: tol must be positive");
  if (max_iter < 1) throw InvalidParameter("fused_solve: max_iter must be at least 1");
  const auto t0 = std::chrono::steady_clock::now();
  Session s(p.m(), p.n(), device);
  s.set_problem(p);
  s.init_col_sums();
  const auto pr = s.iterate(max_iter, tol);
  SolveResult<float> r;
  r.plan = s.plan();
  r.factors = s.factors();
  r.report.solver = "cuda";
  r.report.iterations = pr.iterations;
  r.report.final_error = pr.final_error;
  r.report.converged = pr.converged;
  r.report.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

// fused_iterate (fused.hpp:164-191): `a` and `state` updated in place. Moves
// the matrix over PCIe twice per call; prefer Session for loops.
inline ScalingFactors fused_iterate(Matrix<float>& a, FusedState& state, const Problem<float>& p,
                                    double fi, int device = 0) {
  if (a.rows() != p.m() || a.cols() != p.n())
    throw InvalidParameter("fused_iterate: matrix shape does not match problem");
  if (state.col_sums.size() != a.cols())
    throw InvalidParameter("fused_iterate: carried column sums have wrong length");
  Session s(a.rows(), a.cols(), device);
  Problem<float> cur;
  cur.a = a;
  cur.rpd = p.rpd;
  cur.cpd = p.cpd;
  cur.er = p.er;
  cur.ep = p.ep;
  s.set_problem(cur);
  s.set_fi(fi);
  s.set_state(state);
  s.iterate(1);
  a = s.plan();
  state = s.state();
  return s.factors();
}

// distributed_solve (distributed.hpp:52-130) for rank `rank` of `nranks`
// processes (one per GPU): returns this rank's row block of the plan and alpha,
// the replicated beta, the report and CommStats. nccl_id: 128 bytes from
// uot_nccl_unique_id() on rank 0, shared by the caller's launcher (MPI, torch, ...).
inline DistributedResult<float> distributed_solve(const Problem<float>& p, double tol,
                                                  std::size_t max_iter, int rank, int nranks,
                                                  const std::uint8_t* nccl_id, int device) {
  require_valid(p);
  if (!(tol > 0.0)) throw InvalidParameter("distributed_solve: tol must be positive");
  if (max_iter < 1) throw InvalidParameter("distributed_solve: max_iter must be at least 1");
  const auto t0 = std::chrono::steady_clock::now();
  Session s(p.m(), p.n(), device, rank, nranks, nccl_id);
  const auto lay = s.layout();
  Problem<float> local;
  local.a = Matrix<float>(lay.rows, p.n());
  std::memcpy(local.a.data().data(), p.a.row(lay.row_offset), lay.rows * p.n() * sizeof(float));
  local.rpd.assign(p.rpd.begin() + lay.row_offset, p.rpd.begin() + lay.row_offset + lay.rows);
  local.cpd = p.cpd;
  local.er = p.er;
  local.ep = p.ep;
  s.set_problem(local);
  s.init_col_sums();
  const auto pr = s.iterate(max_iter, tol);
  DistributedResult<float> r;
  r.plan = s.plan();
  r.factors = s.factors();
  r.comm = s.comm();
  r.report.solver = "dist";
  r.report.iterations = pr.iterations;
  r.report.final_error = pr.final_error;
  r.report.converged = pr.converged;
  r.report.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

}  // namespace uot::cuda
