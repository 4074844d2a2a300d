// ref_shim.cpp — C entry points onto the UNMODIFIED reference solver kit.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile together with the
// reference's own sources where they lie under /root/reference/proj/core
// (src/scaling.cpp, src/plan.cpp, src/allreduce.cpp, src/problem_io.cpp) into
// oracle/_ref/libuot_ref.so. Nothing here re-implements the algorithm: each
// function marshals flat buffers into the reference types and calls the
// reference template (fused_solve, fused_iterate_parallel, distributed_solve,
// baseline_solve, gen_problem_t). Used to pin the C restatement
// (oracle/uot_oracle.c), to generate tests/golden/, and as the
// `--impl reference` / cpu_baseline leg of bench.py.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "uot/baseline.hpp"
#include "uot/distributed.hpp"
#include "uot/error.hpp"
#include "uot/fused.hpp"
#include "uot/problem_io.hpp"

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const uot::InvalidParameter& e) {
    g_last_error = e.what();
    return 1;
  } catch (const uot::DegenerateSum& e) {
    g_last_error = e.what();
    return 2;
  } catch (const uot::PartitionError& e) {
    g_last_error = e.what();
    return 3;
  } catch (const uot::IoError& e) {
    g_last_error = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 9;
  }
}

template <typename T>
uot::Problem<T> make_problem(const T* a, std::size_t m, std::size_t n, const double* rpd,
                             const double* cpd, double er, double ep) {
  uot::Problem<T> p;
  p.a = uot::Matrix<T>(m, n);
  std::memcpy(p.a.data().data(), a, m * n * sizeof(T));
  p.rpd.assign(rpd, rpd + m);
  p.cpd.assign(cpd, cpd + n);
  p.er = er;
  p.ep = ep;
  return p;
}

template <typename T>
void copy_out(const uot::Matrix<T>& plan, const uot::ScalingFactors& f, T* plan_out,
              double* alpha, double* beta) {
  if (plan_out) std::memcpy(plan_out, plan.data().data(), plan.size() * sizeof(T));
  if (alpha) std::memcpy(alpha, f.alpha.data(), f.alpha.size() * sizeof(double));
  if (beta) std::memcpy(beta, f.beta.data(), f.beta.size() * sizeof(double));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

int ref_gen_problem_f32(std::uint64_t seed, std::size_t m, std::size_t n, float* a, double* rpd,
                        double* cpd) {
  return guarded([&] {
    const auto p = uot::gen_problem_t<float>(seed, m, n);
    std::memcpy(a, p.a.data().data(), m * n * sizeof(float));
    std::memcpy(rpd, p.rpd.data(), m * sizeof(double));
    std::memcpy(cpd, p.cpd.data(), n * sizeof(double));
  });
}

int ref_compute_fi(double er, double ep, double* fi) {
  return guarded([&] { *fi = uot::compute_fi(er, ep); });
}

int ref_rescale_factor(double t, double s, double fi, double* out) {
  return guarded([&] { *out = uot::rescale_factor(t, s, fi); });
}

int ref_rank_partition(std::size_t ranks, std::size_t rows, std::size_t* bounds) {
  return guarded([&] {
    const auto part = uot::RankPartition::make(ranks, rows);
    bounds[0] = 0;
    for (std::size_t r = 0; r < part.ranks; ++r) bounds[r + 1] = part.blocks[r].end;
  });
}

// fused_solve (fused.hpp:259-285) with WorkerPlan::make(workers).
int ref_fused_solve_f32(const float* a, std::size_t m, std::size_t n, const double* rpd,
                        const double* cpd, double er, double ep, double tol, std::size_t max_iter,
                        std::size_t workers, float* plan_out, double* alpha, double* beta,
                        std::size_t* iterations, double* final_error, int* converged) {
  return guarded([&] {
    const auto p = make_problem(a, m, n, rpd, cpd, er, ep);
    const auto r = uot::fused_solve(p, tol, max_iter, workers);
    copy_out(r.plan, r.factors, plan_out, alpha, beta);
    *iterations = r.report.iterations;
    *final_error = r.report.final_error;
    *converged = r.report.converged ? 1 : 0;
  });
}

int ref_fused_solve_f64(const double* a, std::size_t m, std::size_t n, const double* rpd,
                        const double* cpd, double er, double ep, double tol, std::size_t max_iter,
                        std::size_t workers, double* plan_out, double* alpha, double* beta,
                        std::size_t* iterations, double* final_error, int* converged) {
  return guarded([&] {
    const auto p = make_problem(a, m, n, rpd, cpd, er, ep);
    const auto r = uot::fused_solve(p, tol, max_iter, workers);
    copy_out(r.plan, r.factors, plan_out, alpha, beta);
    *iterations = r.report.iterations;
    *final_error = r.report.final_error;
    *converged = r.report.converged ? 1 : 0;
  });
}

// k calls of fused_iterate_parallel (fused.hpp:197-257) from a block-grouped
// seed (fused.hpp:96-110), exactly like fused_solve's loop without the stop test;
// col_sums receives the carried FusedState.
int ref_fused_iterate_k_f32(const float* a, std::size_t m, std::size_t n, const double* rpd,
                            const double* cpd, double er, double ep, std::size_t workers,
                            std::size_t k, float* plan_out, double* alpha, double* beta,
                            double* col_sums, double* final_error) {
  return guarded([&] {
    const auto p = make_problem(a, m, n, rpd, cpd, er, ep);
    const double fi = uot::compute_fi(er, ep);
    const auto plan = uot::WorkerPlan::make(workers, m, n);
    uot::Matrix<float> x = p.a;
    uot::FusedState st{uot::init_col_sums(x, std::span<const uot::WorkerBlock>(plan.blocks))};
    uot::PartialTable partials(plan.workers, n);
    uot::ScalingFactors f;
    for (std::size_t it = 0; it < k; ++it)
      f = uot::fused_iterate_parallel(x, st, p, fi, plan, partials);
    copy_out(x, f, plan_out, alpha, beta);
    if (col_sums) std::memcpy(col_sums, st.col_sums.data(), n * sizeof(double));
    if (final_error) *final_error = uot::convergence_error(f);
  });
}

// Wall-clock timing of fused_iterate_parallel, seeding and problem setup
// excluded. Returns per-iteration milliseconds in ms_per_iter[k].
// The iteration runs on p.a itself (fused_iterate_parallel reads the Problem
// only for its shape, rpd and cpd: fused.hpp:201-223), so a 16 GiB config-5
// matrix costs one host copy, not two.
int ref_time_fused_iterate_f32(const float* a, std::size_t m, std::size_t n, const double* rpd,
                               const double* cpd, double er, double ep, std::size_t workers,
                               std::size_t k, double* ms_per_iter) {
  return guarded([&] {
    auto p = make_problem(a, m, n, rpd, cpd, er, ep);
    const double fi = uot::compute_fi(er, ep);
    const auto plan = uot::WorkerPlan::make(workers, m, n);
    uot::FusedState st{uot::init_col_sums(p.a, std::span<const uot::WorkerBlock>(plan.blocks))};
    uot::PartialTable partials(plan.workers, n);
    for (std::size_t it = 0; it < k; ++it) {
      const auto t0 = std::chrono::steady_clock::now();
      (void)uot::fused_iterate_parallel(p.a, st, p, fi, plan, partials);
      ms_per_iter[it] =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

// ref_fused_iterate_k_f32 for matrices too large for four host copies (config
// 5: 16 GiB): the caller's buffer `a` receives the plan after k iterations
// (one internal copy; the iteration runs on p.a, see above).
int ref_fused_iterate_k_inplace_f32(float* a, std::size_t m, std::size_t n, const double* rpd,
                                    const double* cpd, double er, double ep, std::size_t workers,
                                    std::size_t k, double* alpha, double* beta, double* col_sums,
                                    double* final_error) {
  return guarded([&] {
    auto p = make_problem(static_cast<const float*>(a), m, n, rpd, cpd, er, ep);
    const double fi = uot::compute_fi(er, ep);
    const auto plan = uot::WorkerPlan::make(workers, m, n);
    uot::FusedState st{uot::init_col_sums(p.a, std::span<const uot::WorkerBlock>(plan.blocks))};
    uot::PartialTable partials(plan.workers, n);
    uot::ScalingFactors f;
    for (std::size_t it = 0; it < k; ++it) f = uot::fused_iterate_parallel(p.a, st, p, fi, plan, partials);
    copy_out(p.a, f, a, alpha, beta);
    if (col_sums) std::memcpy(col_sums, st.col_sums.data(), n * sizeof(double));
    if (final_error) *final_error = uot::convergence_error(f);
  });
}

// distributed_solve (distributed.hpp:52-136).
int ref_distributed_solve_f32(const float* a, std::size_t m, std::size_t n, const double* rpd,
                              const double* cpd, double er, double ep, double tol,
                              std::size_t max_iter, std::size_t ranks, float* plan_out,
                              double* alpha, double* beta, std::size_t* iterations,
                              double* final_error, int* converged, std::uint64_t* allreduce_calls,
                              std::uint64_t* doubles_reduced) {
  return guarded([&] {
    const auto p = make_problem(a, m, n, rpd, cpd, er, ep);
    const auto r = uot::distributed_solve(p, tol, max_iter, ranks);
    copy_out(r.plan, r.factors, plan_out, alpha, beta);
    *iterations = r.report.iterations;
    *final_error = r.report.final_error;
    *converged = r.report.converged ? 1 : 0;
    *allreduce_calls = r.comm.allreduce_calls;
    *doubles_reduced = r.comm.doubles_reduced;
  });
}

// baseline_solve (baseline.hpp:118-142), the reference's 4-pass oracle.
int ref_baseline_solve_f32(const float* a, std::size_t m, std::size_t n, const double* rpd,
                           const double* cpd, double er, double ep, double tol,
                           std::size_t max_iter, float* plan_out, double* alpha, double* beta,
                           std::size_t* iterations, double* final_error, int* converged) {
  return guarded([&] {
    const auto p = make_problem(a, m, n, rpd, cpd, er, ep);
    const auto r = uot::baseline_solve(p, tol, max_iter);
    copy_out(r.plan, r.factors, plan_out, alpha, beta);
    *iterations = r.report.iterations;
    *final_error = r.report.final_error;
    *converged = r.report.converged ? 1 : 0;
  });
}

// write_problem / read_problem (problem_io.cpp:97-141) of a Problem<float>.
int ref_write_problem_f32(const char* path, const float* a, std::size_t m, std::size_t n, const double* rpd,
                          const double* cpd, double er, double ep) {
  return guarded([&] { uot::write_problem(path, uot::AnyProblem(make_problem(a, m, n, rpd, cpd, er, ep))); });
}
int ref_write_problem_f64(const char* path, const double* a, std::size_t m, std::size_t n, const double* rpd,
                          const double* cpd, double er, double ep) {
  return guarded([&] { uot::write_problem(path, uot::AnyProblem(make_problem(a, m, n, rpd, cpd, er, ep))); });
}
// Reads the header (m, n, dtype) and, when the buffers are given, the f32 payload.
int ref_read_problem_f32(const char* path, std::size_t* m, std::size_t* n, int* dtype, double* er, double* ep,
                         float* a, double* rpd, double* cpd) {
  return guarded([&] {
    const uot::AnyProblem any = uot::read_problem(path);
    *m = uot::problem_rows(any);
    *n = uot::problem_cols(any);
    *dtype = uot::problem_dtype(any) == uot::Dtype::f32 ? 1 : 2;
    if (const auto* p = std::get_if<uot::Problem<float>>(&any)) {
      *er = p->er;
      *ep = p->ep;
      if (a) std::memcpy(a, p->a.data().data(), p->a.size() * sizeof(float));
      if (rpd) std::memcpy(rpd, p->rpd.data(), p->rpd.size() * sizeof(double));
      if (cpd) std::memcpy(cpd, p->cpd.data(), p->cpd.size() * sizeof(double));
    } else {
      const auto& q = std::get<uot::Problem<double>>(any);
      *er = q.er;
      *ep = q.ep;
    }
  });
}

}  // extern "C"
