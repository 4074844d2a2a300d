// uot/cuda.hpp — drop-in B200 backend for the reference solver API.
//
// Header-only C++ facade over the C ABI (include/uot_cuda.h). It is written
// against the reference's own types and exceptions
// (/root/reference/proj/core/include/uot: Problem<T>, Matrix<T>, FusedState,
// ScalingFactors, SolveResult<T>, DistributedResult<T>, InvalidParameter,
// DegenerateSum, PartitionError, ConfigError), so a reference user switches a
// call site by changing the namespace:
//
//   uot::fused_solve(p, tol, max_iter[, workers]) ->  uot::cuda::fused_solve(p, tol, max_iter[, workers])
//   uot::fused_solve(p, tol, max_iter, plan)      ->  uot::cuda::fused_solve(p, tol, max_iter, plan)
//   uot::fused_iterate(a, state, p, fi)           ->  uot::cuda::fused_iterate(a, state, p, fi)
//   uot::fused_iterate_parallel(a, st, p, fi, plan[, partials]) -> uot::cuda::fused_iterate_parallel(same)
//   uot::distributed_solve(p, tol, max_iter, P)   ->  uot::cuda::distributed_solve(p, tol, max_iter, P)  (one process,
//                                                     every rank on a GPU), or one process per GPU:
//                                                     uot::cuda::distributed_solve(p, tol, max_iter, rank, P, nccl_id)
//                                                     or uot::cuda::distributed_solve_peer(..., allgather)
//   uot::baseline_solve(p, tol, max_iter)         ->  uot::cuda::baseline_solve(p, tol, max_iter)
//   uot::tiled_solve(p, tol, max_iter, ...)       ->  uot::cuda::tiled_solve(p, tol, max_iter)
//   uot::read_problem(path) + solve               ->  uot::cuda::load(path).iterate(...)
//
// An integral 4th argument of fused_solve means workers everywhere, as in the
// reference (fused.hpp:287-291); the GPU is chosen with a trailing
// uot::cuda::Device{n} (default: device 0), never by a bare integer.
//
// plus uot::cuda::Session for loops that should keep the matrix resident in HBM
// (the reference's per-iteration API moves the whole matrix every call).
// Include the reference headers first (uot/problem.hpp, uot/fused.hpp,
// uot/distributed.hpp) and link libuot_cuda.so. See INTEGRATION.md.
#pragma once

#include <array>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <functional>
#include <memory>
#include <span>
#include <string>
#include <type_traits>
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
    case UOT_IO_ERROR: throw IoError(what);
    default: throw Error("cuda backend: " + what);
  }
}

// The GPU a solver call runs on. A distinct type so that an integer argument in
// a reference call site keeps its reference meaning (workers, ranks, ...).
struct Device {
  int id = 0;
  constexpr Device() = default;
  constexpr explicit Device(int i) : id(i) {}
};

// A problem resident on one B200 (or one rank's row block of it).
class Session {
 public:
  Session(std::size_t rows, std::size_t cols, int device = 0, Dtype dtype = Dtype::f32) {
    check(uot_create(&ctx_, rows, cols, dtype == Dtype::f64 ? UOT_F64 : UOT_F32, device));
  }
  // Rank `rank` of `nranks`, rows split by RankPartition::make (plan.cpp:35-44).
  Session(std::size_t global_rows, std::size_t cols, int device, int rank, int nranks,
          const std::uint8_t* nccl_id) {
    check(uot_create_dist(&ctx_, global_rows, cols, UOT_F32, device, rank, nranks, nccl_id));
  }
  // Rank `rank` of `nranks` whose per-iteration allreduce is fused into the
  // finalize kernels over peer memory (CUDA IPC over NVLink): connect() with
  // every rank's peer_handle() before use (uot_create_peer, include/uot_cuda.h).
  struct Peer {};
  Session(std::size_t global_rows, std::size_t cols, int device, int rank, int nranks, Peer) {
    check(uot_create_peer(&ctx_, global_rows, cols, UOT_F32, device, rank, nranks));
  }
  std::array<std::uint8_t, 64> peer_handle() const {
    std::array<std::uint8_t, 64> h{};
    check(uot_peer_handle(ctx_, h.data()));
    return h;
  }
  void connect(const std::vector<std::array<std::uint8_t, 64>>& handles) {
    std::vector<std::uint8_t> flat;
    for (const auto& h : handles) flat.insert(flat.end(), h.begin(), h.end());
    check(uot_peer_connect(ctx_, flat.data()));
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
  // Problem<double> (Dtype::f64 session): plain f64 products, as fused.hpp:128-140 with T = double.
  void set_problem(const Problem<double>& p) {
    check(uot_set_problem_f64(ctx_, p.a.data().data(), p.rpd.data(), p.cpd.data(), p.er, p.ep));
  }
  void set_plan(const Matrix<double>& a) { check(uot_set_plan_f64(ctx_, a.data().data())); }
  Matrix<double> plan_f64() const {
    Matrix<double> m(rows(), cols());
    check(uot_get_plan_f64(ctx_, m.data().data()));
    return m;
  }
  Dtype dtype() const { return layout().dtype == UOT_F64 ? Dtype::f64 : Dtype::f32; }
  void set_fi(double fi) { check(uot_set_fi(ctx_, fi)); }
  // read_problem / write_problem (problem_io.cpp:97-141) of this session's rows,
  // streamed between the .uotp file and HBM.
  void load_problem_file(const std::filesystem::path& path) { check(uot_load_problem_file(ctx_, path.c_str())); }
  void save_problem_file(const std::filesystem::path& path) const {
    check(uot_save_problem_file(ctx_, path.c_str()));
  }
  // UOT_VARIANT_FUSED (default), UOT_VARIANT_TWO_PASS (tiled.hpp), UOT_VARIANT_BASELINE (baseline.hpp).
  void set_variant(int variant) { check(uot_set_variant(ctx_, variant)); }
  void set_deterministic(bool on) { check(uot_set_deterministic(ctx_, on ? 1 : 0)); }
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
  // The plan into an existing rows() x cols() matrix (no reallocation).
  void plan_into(Matrix<float>& m) const { check(uot_get_plan(ctx_, m.data().data())); }
  void plan_into(Matrix<double>& m) const { check(uot_get_plan_f64(ctx_, m.data().data())); }
  // fused_iterate's inputs as given (fused.hpp:164-191): the current plan, the
  // marginals and fi, uploaded without require_valid's checks.
  template <typename T>
  void set_iterate_input(const Matrix<T>& a, const std::vector<double>& rpd, const std::vector<double>& cpd,
                         double fi) {
    check(uot_set_iterate_input(ctx_, a.data().data(), std::is_same_v<T, double> ? UOT_F64 : UOT_F32, rpd.data(),
                                cpd.data(), fi));
  }
  // set_problem from the pieces, without assembling a Problem (no host copy of a).
  void set_problem(const Matrix<float>& a, const std::vector<double>& rpd, const std::vector<double>& cpd,
                   double er, double ep) {
    check(uot_set_problem(ctx_, a.data().data(), rpd.data(), cpd.data(), er, ep));
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

// fused_solve (fused.hpp:259-285) on one B200, for Problem<float> or
// Problem<double>. The plan, factors and report have the reference's meaning;
// report.solver is "cuda" and wall_ms also covers the PCIe transfers.
template <typename T>
inline SolveResult<T> fused_solve(const Problem<T>& p, double tol, std::size_t max_iter, Device device = Device{}) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "Problem<float> or Problem<double>");
  require_valid(p);
  if (!(tol > 0.0)) throw InvalidParameter("fused_solve: tol must be positive");
  if (max_iter < 1) throw InvalidParameter("fused_solve: max_iter must be at least 1");
  const auto t0 = std::chrono::steady_clock::now();
  Session s(p.m(), p.n(), device.id, std::is_same_v<T, double> ? Dtype::f64 : Dtype::f32);
  s.set_problem(p);
  s.init_col_sums();
  const auto pr = s.iterate(max_iter, tol);
  SolveResult<T> r;
  if constexpr (std::is_same_v<T, double>)
    r.plan = s.plan_f64();
  else
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

// fused_solve(p, tol, max_iter, std::size_t workers) (fused.hpp:287-291). Any
// integral 4th argument binds here and means workers, as in the reference
// (uot::cuda::fused_solve(p, tol, 200, 8) is 8 workers, not GPU 8). The worker
// count is a host-thread knob with no GPU meaning (results match any W to the
// parity bar); it is validated like WorkerPlan::make validates it.
template <typename T, typename W, std::enable_if_t<std::is_integral_v<W> && !std::is_same_v<W, bool>, int> = 0>
inline SolveResult<T> fused_solve(const Problem<T>& p, double tol, std::size_t max_iter, W workers,
                                  Device device = Device{}) {
  if (workers < W(1)) throw InvalidParameter("fused_solve: workers must be at least 1");
  return uot::cuda::fused_solve<T>(p, tol, max_iter, device);
}

// fused_solve(p, tol, max_iter, const WorkerPlan&) (fused.hpp:259-285): the
// reference's host worker plan has no GPU meaning — the sweep's CTA schedule
// replaces it — but it is validated like the reference validates it, so a call
// site switches by namespace alone. Results match any worker count to the
// parity bar (the reference's own W-independence, test_fused.cpp).
template <typename T>
inline SolveResult<T> fused_solve(const Problem<T>& p, double tol, std::size_t max_iter, const WorkerPlan& plan,
                                  Device device = Device{}) {
  if (plan.blocks.empty() || plan.blocks.back().end != p.m())
    throw InvalidParameter("fused_solve: plan does not cover the matrix rows");
  return uot::cuda::fused_solve<T>(p, tol, max_iter, device);
}

namespace detail {
template <typename T>
inline SolveResult<T> solve_with(const Problem<T>& p, double tol, std::size_t max_iter, Device device, int variant,
                                 const char* solver, const char* who) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "Problem<float> or Problem<double>");
  require_valid(p);
  if (!(tol > 0.0)) throw InvalidParameter(std::string(who) + ": tol must be positive");
  if (max_iter < 1) throw InvalidParameter(std::string(who) + ": max_iter must be at least 1");
  const auto t0 = std::chrono::steady_clock::now();
  Session s(p.m(), p.n(), device.id, std::is_same_v<T, double> ? Dtype::f64 : Dtype::f32);
  s.set_problem(p);
  s.init_col_sums();
  s.set_variant(variant);
  const auto pr = s.iterate(max_iter, tol);
  SolveResult<T> r;
  if constexpr (std::is_same_v<T, double>)
    r.plan = s.plan_f64();
  else
    r.plan = s.plan();
  r.factors = s.factors();
  r.report.solver = solver;
  r.report.iterations = pr.iterations;
  r.report.final_error = pr.final_error;
  r.report.converged = pr.converged;
  r.report.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return r;
}
}  // namespace detail

// baseline_solve (baseline.hpp:118-142): the four-sweep schedule on the GPU
// (an ablation of the fused sweep: 3x its HBM traffic).
template <typename T>
inline SolveResult<T> baseline_solve(const Problem<T>& p, double tol, std::size_t max_iter,
                                     Device device = Device{}) {
  return detail::solve_with(p, tol, max_iter, device, UOT_VARIANT_BASELINE, "baseline", "baseline_solve");
}

// tiled_solve (tiled.hpp:231-260): the paper's two-pass GPU data flow (part4 ->
// row factors -> part2); the reference's TileConfig shapes have no meaning here.
template <typename T>
inline SolveResult<T> tiled_solve(const Problem<T>& p, double tol, std::size_t max_iter, Device device = Device{}) {
  return detail::solve_with(p, tol, max_iter, device, UOT_VARIANT_TWO_PASS, "tiled", "tiled_solve");
}

// A session holding the problem of a .uotp file (read_problem, problem_io.cpp:106-141).
inline Session load(const std::filesystem::path& path, Device device = Device{}) {
  std::uint64_t m = 0, n = 0;
  int dtype = 0;
  double er = 0, ep = 0;
  const int rc = uot_problem_file_info(path.c_str(), &m, &n, &dtype, &er, &ep);
  if (rc != UOT_OK) raise(rc, uot_last_io_error());
  Session s(m, n, device.id, dtype == UOT_F64 ? Dtype::f64 : Dtype::f32);
  s.load_problem_file(path);
  return s;
}

// fused_iterate (fused.hpp:164-191) for Problem<float> or Problem<double>: `a`
// and `state` updated in place. Like the reference it takes fi and the plan as
// given — no require_valid, no positivity check of the current plan — and
// throws DegenerateSum where beta_from_state / rescale_factor would. Moves the
// matrix over PCIe twice per call; prefer Session for loops.
template <typename T>
inline ScalingFactors fused_iterate(Matrix<T>& a, FusedState& state, const Problem<T>& p, double fi,
                                    Device device = Device{}) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "Matrix<float> or Matrix<double>");
  if (a.rows() != p.m() || a.cols() != p.n())
    throw InvalidParameter("fused_iterate: matrix shape does not match problem");
  if (state.col_sums.size() != a.cols())
    throw InvalidParameter("fused_iterate: carried column sums have wrong length");
  // One device session per thread, shape and dtype, kept between calls: a loop
  // over fused_iterate pays the two PCIe transfers per call, not a session setup.
  thread_local std::unique_ptr<Session> cached;
  thread_local std::size_t cr = 0, cc = 0;
  thread_local int cd = -1;
  if (!cached || cr != a.rows() || cc != a.cols() || cd != device.id) {
    cached.reset();
    cached = std::make_unique<Session>(a.rows(), a.cols(), device.id,
                                       std::is_same_v<T, double> ? Dtype::f64 : Dtype::f32);
    cr = a.rows(), cc = a.cols(), cd = device.id;
  }
  Session& s = *cached;
  s.set_iterate_input(a, p.rpd, p.cpd, fi);
  s.set_state(state);
  s.iterate(1);
  s.plan_into(a);
  state = s.state();
  return s.factors();
}

// fused_iterate_parallel (fused.hpp:197-257) with the reference's checks on the
// plan and partial table; the GPU does the iteration (fused_iterate above).
template <typename T>
inline ScalingFactors fused_iterate_parallel(Matrix<T>& a, FusedState& state, const Problem<T>& p, double fi,
                                             const WorkerPlan& plan, PartialTable& partials,
                                             Device device = Device{}) {
  if (a.rows() != p.m() || a.cols() != p.n())
    throw InvalidParameter("fused_iterate_parallel: matrix shape does not match problem");
  if (state.col_sums.size() != a.cols())
    throw InvalidParameter("fused_iterate_parallel: carried column sums have wrong length");
  if (plan.blocks.empty() || plan.blocks.back().end != a.rows())
    throw InvalidParameter("fused_iterate_parallel: plan does not cover the matrix rows");
  if (partials.workers() < plan.workers || partials.cols() != a.cols())
    throw InvalidParameter("fused_iterate_parallel: partial table does not fit the plan");
  return uot::cuda::fused_iterate<T>(a, state, p, fi, device);
}
template <typename T>
inline ScalingFactors fused_iterate_parallel(Matrix<T>& a, FusedState& state, const Problem<T>& p, double fi,
                                             const WorkerPlan& plan, Device device = Device{}) {
  PartialTable partials(plan.workers, a.cols());
  return uot::cuda::fused_iterate_parallel<T>(a, state, p, fi, plan, partials, device);
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

// distributed_solve with the column-sum allreduce fused into the finalize
// kernels over peer memory: `allgather` is the caller's transport (MPI,
// torch.distributed, a shared file, ...) and must return every rank's 64-byte
// handle in rank order.
using AllGather = std::function<std::vector<std::array<std::uint8_t, 64>>(const std::array<std::uint8_t, 64>&)>;
inline DistributedResult<float> distributed_solve_peer(const Problem<float>& p, double tol, std::size_t max_iter,
                                                       int rank, int nranks, int device, const AllGather& allgather) {
  require_valid(p);
  if (!(tol > 0.0)) throw InvalidParameter("distributed_solve: tol must be positive");
  if (max_iter < 1) throw InvalidParameter("distributed_solve: max_iter must be at least 1");
  const auto t0 = std::chrono::steady_clock::now();
  Session s(p.m(), p.n(), device, rank, nranks, Session::Peer{});
  if (nranks > 1) s.connect(allgather(s.peer_handle()));
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

// distributed_solve(p, tol, max_iter, RankPartition | ranks) (distributed.hpp:52-142)
// with the reference's own signature: every rank in THIS process
// (uot_create_group), rank r on GPU r mod (visible GPUs), one fused peer-memory
// exchange of the column sums per iteration; the whole plan and alpha come back,
// as in the reference. Blocks must be contiguous and non-empty.
template <typename T>
inline DistributedResult<T> distributed_solve(const Problem<T>& p, double tol, std::size_t max_iter,
                                              const RankPartition& part) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "Problem<float> or Problem<double>");
  constexpr bool kF64 = std::is_same_v<T, double>;
  require_valid(p);
  if (!(tol > 0.0)) throw InvalidParameter("distributed_solve: tol must be positive");
  if (max_iter < 1) throw InvalidParameter("distributed_solve: max_iter must be at least 1");
  const std::size_t m = p.m(), n = p.n(), R = part.ranks;
  if (part.blocks.size() != R || part.blocks.empty() || part.blocks.back().end != m)
    throw PartitionError("distributed_solve: partition does not cover the matrix rows");
  std::vector<std::uint64_t> bounds(R + 1, 0);
  for (std::size_t r = 0; r < R; ++r) {
    if (part.blocks[r].begin != bounds[r]) throw PartitionError("distributed_solve: partition blocks are not contiguous");
    bounds[r + 1] = part.blocks[r].end;
  }
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<uot_ctx*> ctx(R, nullptr);
  struct Guard {
    std::vector<uot_ctx*>& c;
    ~Guard() {
      for (auto* x : c) uot_destroy(x);
    }
  } guard{ctx};
  auto fail = [&](int rc) {
    std::string msg = "session group";
    for (auto* x : ctx)
      if (x && *uot_last_error(x)) msg = uot_last_error(x);
    raise(rc, msg);
  };
  int rc = uot_create_group(ctx.data(), m, n, kF64 ? UOT_F64 : UOT_F32, nullptr, static_cast<int>(R), bounds.data());
  if (rc) fail(rc);
  for (std::size_t r = 0; r < R; ++r) {
    const std::size_t b = bounds[r];
    if constexpr (kF64)
      rc = uot_set_problem_f64(ctx[r], p.a.row(b), p.rpd.data() + b, p.cpd.data(), p.er, p.ep);
    else
      rc = uot_set_problem(ctx[r], p.a.row(b), p.rpd.data() + b, p.cpd.data(), p.er, p.ep);
    if (rc) fail(rc);
  }
  if ((rc = uot_group_init_col_sums(ctx.data(), static_cast<int>(R)))) fail(rc);
  std::uint64_t it = 0;
  double err = 0.0;
  int conv = 0;
  if ((rc = uot_group_iterate(ctx.data(), static_cast<int>(R), max_iter, tol, &it, &err, &conv))) fail(rc);
  DistributedResult<T> out;
  out.plan = Matrix<T>(m, n);
  out.factors.alpha.resize(m);
  out.factors.beta.resize(n);
  for (std::size_t r = 0; r < R; ++r) {
    const std::size_t b = bounds[r];
    if constexpr (kF64)
      rc = uot_get_plan_f64(ctx[r], out.plan.row(b));
    else
      rc = uot_get_plan(ctx[r], out.plan.row(b));
    if (rc) fail(rc);
    if ((rc = uot_get_factors(ctx[r], out.factors.alpha.data() + b, r == 0 ? out.factors.beta.data() : nullptr)))
      fail(rc);
  }
  out.comm.allreduce_calls = it;  // one exchange of the column vector per iteration (distributed.hpp:88-94)
  out.comm.doubles_reduced = it * n;
  out.report.solver = "dist";
  out.report.iterations = it;
  out.report.final_error = err;
  out.report.converged = conv != 0;
  out.report.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return out;
}
template <typename T>
inline DistributedResult<T> distributed_solve(const Problem<T>& p, double tol, std::size_t max_iter,
                                              std::size_t ranks) {
  return uot::cuda::distributed_solve<T>(p, tol, max_iter, RankPartition::make(ranks, p.m()));
}

}  // namespace uot::cuda
