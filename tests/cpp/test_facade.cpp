// C++ parity suite for the drop-in facade (include/uot/cuda.hpp), written like
// the reference's own doctest suites (proj/tests/test_fused.cpp,
// test_distributed.cpp) but against the CUDA backend. It links the UNMODIFIED
// reference (oracle/_ref, compiled from /root/reference) as the oracle, so it
// is test infrastructure: built by oracle/Makefile into oracle/_ref/test_facade
// and run on the GPU box by tests/test_gpu_facade.py. Exit code = failures.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "uot/baseline.hpp"
#include "uot/cuda.hpp"
#include "uot/fused.hpp"
#include "uot/problem_io.hpp"
#include "uot/tiled.hpp"

namespace {

int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(cond)) {                                                        \
      ++g_fail;                                                           \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    bool ok_ = false;                                                     \
    try {                                                                 \
      (void)(expr);                                                       \
    } catch (const T&) {                                                  \
      ok_ = true;                                                         \
    } catch (...) {                                                       \
    }                                                                     \
    if (!ok_) {                                                           \
      ++g_fail;                                                           \
      std::fprintf(stderr, "%s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                     \
  } while (0)

constexpr double kNever = 1e-300;

uot::Problem<float> random_problem(std::uint64_t seed, std::size_t m, std::size_t n, double fi) {
  auto p = uot::gen_problem_t<float>(seed, m, n);  // oracle.hpp:61-67
  p.er = 1.0;
  p.ep = (1.0 - fi) / fi;
  return p;
}

double max_rel(const uot::Matrix<float>& a, const uot::Matrix<float>& b) {
  double m = 0.0;
  for (std::size_t k = 0; k < a.size(); ++k)
    m = std::max(m, std::abs(double(a.data()[k]) - double(b.data()[k])) / std::abs(double(b.data()[k])));
  return m;
}

void test_solve_matches_reference() {
  struct C { std::uint64_t seed; std::size_t m, n; double fi; std::size_t k, w; };
  for (const C c : {C{21, 16, 16, 0.5, 25, 1}, C{22, 10, 33, 1.0, 25, 1}, C{33, 128, 128, 0.5, 100, 4},
                    C{42, 1024, 1024, 1 / 1.1, 100, 8}, C{5, 300, 20000, 1 / 1.1, 10, 8}}) {
    const auto p = random_problem(c.seed, c.m, c.n, c.fi);
    const auto ref = uot::fused_solve(p, kNever, c.k, c.w);
    const auto gpu = uot::cuda::fused_solve(p, kNever, c.k);
    CHECK(gpu.report.iterations == c.k);
    CHECK(max_rel(gpu.plan, ref.plan) <= 1e-5);
    CHECK(gpu.plan == ref.plan);  // same arithmetic: bit-identical
    CHECK(std::abs(gpu.report.final_error - ref.report.final_error) <= 1e-5 * ref.report.final_error);
    CHECK(uot::max_abs_diff(gpu.factors.alpha, ref.factors.alpha) <= 1e-12);
    CHECK(uot::max_abs_diff(gpu.factors.beta, ref.factors.beta) <= 1e-12);
  }
}

void test_hand_checked_iteration() {  // test_fused.cpp:38-56 in fp32
  uot::Problem<float> p;
  p.a = uot::Matrix<float>{{1.f, 1.f}, {1.f, 1.f}};
  p.rpd = {4.0, 2.0};
  p.cpd = {3.0, 3.0};
  uot::Matrix<float> a = p.a;
  uot::FusedState st{uot::init_col_sums(a)};
  const auto f = uot::cuda::fused_iterate(a, st, p, 1.0);
  CHECK(f.beta == std::vector<double>({1.5, 1.5}));
  CHECK(std::abs(f.alpha[0] - 4.0 / 3.0) <= 1e-15);
  CHECK(std::abs(f.alpha[1] - 2.0 / 3.0) <= 1e-15);
  CHECK(a(0, 0) == 2.f && a(1, 1) == 1.f);
  CHECK(std::abs(st.col_sums[0] - 3.0) <= 1e-14);
  CHECK(std::abs(uot::convergence_error(f) - 0.5) <= 1e-15);
}

void test_per_iteration_api_tracks_reference() {
  const auto p = random_problem(31, 64, 96, 0.5);
  uot::Matrix<float> mine = p.a, theirs = p.a;
  uot::FusedState sm{uot::init_col_sums(mine)}, st{uot::init_col_sums(theirs)};
  for (int it = 0; it < 6; ++it) {
    const auto fm = uot::cuda::fused_iterate(mine, sm, p, 0.5);
    const auto ft = uot::fused_iterate(theirs, st, p, 0.5);
    CHECK(uot::max_abs_diff(fm.alpha, ft.alpha) <= 1e-13);
  }
  CHECK(mine == theirs);
}

void test_session_is_resumable_and_converges() {
  auto p = random_problem(37, 24, 24, 0.5);
  double sr = 0, sc = 0;
  for (double v : p.rpd) sr += v;
  for (double v : p.cpd) sc += v;
  for (double& v : p.cpd) v *= sr / sc;  // balanced_problem (oracle.hpp:74-83)
  const auto ref = uot::fused_solve(p, 1e-6, 10000);
  uot::cuda::Session s(24, 24);
  s.set_problem(p);
  s.init_col_sums();
  std::size_t total = 0;
  bool conv = false;
  while (!conv && total < 10000) {
    const auto pr = s.iterate(7, 1e-6);
    total += pr.iterations;
    conv = pr.converged;
  }
  CHECK(ref.report.converged && conv);
  CHECK(total == ref.report.iterations);
  CHECK(max_rel(s.plan(), ref.plan) <= 1e-5);
}

void test_errors_map_to_reference_exceptions() {
  const auto p = random_problem(38, 4, 4, 0.5);
  CHECK_THROWS_AS(uot::cuda::fused_solve(p, 0.0, 10), uot::InvalidParameter);
  CHECK_THROWS_AS(uot::cuda::fused_solve(p, 1e-6, 0), uot::InvalidParameter);
  uot::Matrix<float> a = p.a;
  uot::FusedState zero{std::vector<double>(4, 0.0)};
  CHECK_THROWS_AS(uot::cuda::fused_iterate(a, zero, p, 0.5), uot::DegenerateSum);
  uot::FusedState bad_len{std::vector<double>(3, 1.0)};
  CHECK_THROWS_AS(uot::cuda::fused_iterate(a, bad_len, p, 0.5), uot::InvalidParameter);
  auto broken = p;
  broken.a(0, 0) = -1.f;
  CHECK_THROWS_AS(uot::cuda::fused_solve(broken, 1e-6, 10), uot::InvalidParameter);
  std::uint8_t id[128] = {0};
  CHECK_THROWS_AS(uot::cuda::distributed_solve(p, 1e-6, 10, 0, 5, id, 0), uot::PartitionError);
}

void test_single_rank_distributed() {  // test_distributed.cpp:92-104, 142-155
  const auto p = random_problem(24, 64, 64, 0.5);
  // a real id: with one rank and an id the session runs the NCCL exchange path
  // (a one-rank communicator, ncclAllReduce per iteration)
  std::uint8_t id[128] = {0};
  CHECK(uot_nccl_unique_id(id) == UOT_OK);
  const auto d = uot::cuda::distributed_solve(p, kNever, 37, 0, 1, id, 0);
  const auto ref = uot::distributed_solve(p, kNever, 37, std::size_t(1));
  CHECK(d.report.iterations == 37 && d.report.solver == "dist");
  CHECK(d.comm.allreduce_calls == 37 && d.comm.doubles_reduced == 37u * 64u);
  CHECK(max_rel(d.plan, ref.plan) <= 1e-5);
}

void test_ablation_solvers_match_reference() {  // baseline.hpp:118-142, tiled.hpp
  const auto p = random_problem(9, 200, 300, 0.5);
  const auto rb = uot::baseline_solve(p, kNever, 12);
  const auto gb = uot::cuda::baseline_solve(p, kNever, 12);
  CHECK(gb.report.iterations == 12 && gb.report.solver == "baseline");
  CHECK(max_rel(gb.plan, rb.plan) <= 1e-5);
  CHECK(std::abs(gb.report.final_error - rb.report.final_error) <= 1e-9 * rb.report.final_error);
  const auto rt = uot::tiled_solve(p, kNever, 12, uot::default_part2_config(200, 300), uot::default_part4_config(200, 300));
  const auto gt = uot::cuda::tiled_solve(p, kNever, 12);
  CHECK(max_rel(gt.plan, rt.plan) <= 1e-5);
}

void test_problem_files_round_trip() {  // problem_io.cpp:97-141
  const auto p = random_problem(13, 40, 70, 0.5);
  const std::filesystem::path in = std::filesystem::temp_directory_path() / "uot_facade_in.uotp";
  const std::filesystem::path out = std::filesystem::temp_directory_path() / "uot_facade_out.uotp";
  uot::write_problem(in, uot::AnyProblem(p));
  auto s = uot::cuda::load(in);
  CHECK(s.plan() == p.a);
  s.init_col_sums();
  s.iterate(5);
  s.save_problem_file(out);
  const auto back = std::get<uot::Problem<float>>(uot::read_problem(out));
  const auto ref = uot::fused_solve(p, kNever, 5);
  CHECK(max_rel(back.a, ref.plan) <= 1e-5);
  CHECK(back.rpd == p.rpd && back.cpd == p.cpd && back.er == p.er && back.ep == p.ep);
  CHECK_THROWS_AS(uot::cuda::load("/nonexistent/uot/path.uotp"), uot::IoError);
  std::filesystem::remove(in);
  std::filesystem::remove(out);
}

void test_f64_problem_matches_reference() {  // Problem<double>, Dtype::f64
  auto p = uot::gen_problem_t<double>(44, 300, 700);
  p.er = 1.0;
  p.ep = 0.25;
  const auto ref = uot::fused_solve(p, kNever, 15, std::size_t(4));
  const auto gpu = uot::cuda::fused_solve(p, kNever, 15);
  CHECK(gpu.report.iterations == 15);
  double m = 0.0;
  for (std::size_t k = 0; k < gpu.plan.size(); ++k)
    m = std::max(m, std::abs(gpu.plan.data()[k] - ref.plan.data()[k]) / ref.plan.data()[k]);
  CHECK(m <= 1e-12);
  CHECK(uot::max_abs_diff(gpu.factors.beta, ref.factors.beta) <= 1e-12);
  const auto rb = uot::baseline_solve(p, kNever, 7);  // the f64 ablations (baseline.hpp / tiled.hpp, T = double)
  const auto gb = uot::cuda::baseline_solve(p, kNever, 7);
  const auto gt = uot::cuda::tiled_solve(p, kNever, 7);
  const auto rt = uot::fused_solve(p, kNever, 7, std::size_t(2));
  double mb = 0.0, mt = 0.0;
  for (std::size_t k = 0; k < gb.plan.size(); ++k) {
    mb = std::max(mb, std::abs(gb.plan.data()[k] - rb.plan.data()[k]) / rb.plan.data()[k]);
    mt = std::max(mt, std::abs(gt.plan.data()[k] - rt.plan.data()[k]) / rt.plan.data()[k]);
  }
  CHECK(gb.report.iterations == 7 && mb <= 1e-12);
  CHECK(gt.report.iterations == 7 && mt <= 1e-12);
}

void test_single_rank_peer_distributed() {
  const auto p = random_problem(25, 64, 64, 0.5);
  const auto d = uot::cuda::distributed_solve_peer(p, kNever, 11, 0, 1, 0,
                                                   [](const std::array<std::uint8_t, 64>& h) {
                                                     return std::vector<std::array<std::uint8_t, 64>>{h};
                                                   });
  const auto ref = uot::distributed_solve(p, kNever, 11, std::size_t(1));
  CHECK(d.report.iterations == 11 && max_rel(d.plan, ref.plan) <= 1e-5);
}

void test_in_process_ranks_match_reference() {  // test_distributed.cpp:106-118, one process, reference signature
  const auto p = random_problem(26, 301, 2000, 0.5);
  for (std::size_t ranks : {std::size_t(2), std::size_t(3)}) {
    const auto d = uot::cuda::distributed_solve(p, kNever, 9, ranks);
    const auto ref = uot::distributed_solve(p, kNever, 9, ranks);
    CHECK(d.report.iterations == 9 && d.report.solver == "dist");
    CHECK(d.comm.allreduce_calls == ref.comm.allreduce_calls && d.comm.doubles_reduced == ref.comm.doubles_reduced);
    CHECK(max_rel(d.plan, ref.plan) <= 1e-5);
    CHECK(uot::max_abs_diff(d.factors.beta, ref.factors.beta) <= 1e-12);
    CHECK(std::abs(d.report.final_error - ref.report.final_error) <= 1e-9 * std::max(1.0, ref.report.final_error));
  }
  uot::RankPartition gap;
  gap.ranks = 2;
  gap.blocks = {{0, 100}, {150, 301}};
  CHECK_THROWS_AS(uot::cuda::distributed_solve(p, kNever, 3, gap), uot::PartitionError);
  CHECK_THROWS_AS(uot::cuda::distributed_solve(p, kNever, 3, std::size_t(302)), uot::PartitionError);
}

void test_worker_plan_overloads() {  // fused.hpp:197-208, 259-285: same call shapes and checks
  const auto p = random_problem(27, 120, 500, 0.5);
  const auto plan = uot::WorkerPlan::make(4, p.m(), p.n());
  const auto ref = uot::fused_solve(p, kNever, 6, plan);
  const auto gpu = uot::cuda::fused_solve(p, kNever, 6, plan);
  CHECK(gpu.report.iterations == 6 && max_rel(gpu.plan, ref.plan) <= 1e-5);
  uot::Matrix<float> ra = p.a, ga = p.a;
  uot::FusedState rs{uot::init_col_sums(ra)}, gs{uot::init_col_sums(ga)};
  const double fi = uot::compute_fi(p.er, p.ep);
  for (int it = 0; it < 3; ++it) {
    const auto rf = uot::fused_iterate_parallel(ra, rs, p, fi, plan);
    const auto gf = uot::cuda::fused_iterate_parallel(ga, gs, p, fi, plan);
    CHECK(uot::max_abs_diff(rf.beta, gf.beta) <= 1e-12);
  }
  CHECK(max_rel(ga, ra) <= 1e-5);
  uot::WorkerPlan bad = plan;
  bad.blocks.back().end -= 1;
  CHECK_THROWS_AS(uot::cuda::fused_solve(p, kNever, 2, bad), uot::InvalidParameter);
  CHECK_THROWS_AS(uot::cuda::fused_iterate_parallel(ga, gs, p, fi, bad), uot::InvalidParameter);
  uot::PartialTable small(1, p.n());
  CHECK_THROWS_AS(uot::cuda::fused_iterate_parallel(ga, gs, p, fi, plan, small), uot::InvalidParameter);
}

void test_integral_fourth_argument_means_workers() {  // fused.hpp:287-291 call shapes
  // uot::fused_solve(p, tol, it, 8) is 8 workers; switched by namespace it must
  // stay 8 workers on device 0 (a one-GPU box has no device 8), for every
  // integral type a call site may pass.
  const auto p = random_problem(28, 96, 130, 0.5);
  const auto ref = uot::fused_solve(p, kNever, 10, 8);
  const auto a = uot::cuda::fused_solve(p, kNever, 10, 8);
  const auto b = uot::cuda::fused_solve(p, kNever, 10, 8u);
  const auto c = uot::cuda::fused_solve(p, kNever, 10, 8L);
  const auto d = uot::cuda::fused_solve(p, kNever, 10, std::size_t(8));
  const auto e = uot::cuda::fused_solve(p, kNever, 10, uot::cuda::Device{0});
  const auto f = uot::cuda::fused_solve(p, kNever, 10, 3, uot::cuda::Device{0});
  for (const auto* r : {&a, &b, &c, &d, &e, &f}) {
    CHECK(r->report.iterations == 10);
    CHECK(max_rel(r->plan, ref.plan) <= 1e-5);
  }
  CHECK(a.plan == b.plan && a.plan == d.plan && a.plan == e.plan);
  CHECK_THROWS_AS(uot::cuda::fused_solve(p, kNever, 10, 0), uot::InvalidParameter);
  CHECK_THROWS_AS(uot::cuda::fused_solve(p, kNever, 10, -2), uot::InvalidParameter);
}

void test_fused_iterate_takes_inputs_as_given() {  // fused.hpp:164-191: shape checks only
  // a zero plan entry and an unvalidated Problem (ep < 0 would fail
  // require_valid) iterate exactly like the reference's fused_iterate
  auto p = random_problem(29, 40, 64, 0.5);
  p.ep = -0.5;
  uot::Matrix<float> mine = p.a, theirs = p.a;
  mine(3, 5) = theirs(3, 5) = 0.f;
  uot::FusedState sm{uot::init_col_sums(mine)}, st{uot::init_col_sums(theirs)};
  for (int it = 0; it < 4; ++it) {
    const auto fm = uot::cuda::fused_iterate(mine, sm, p, 0.7);
    const auto ft = uot::fused_iterate(theirs, st, p, 0.7);
    CHECK(uot::max_abs_diff(fm.alpha, ft.alpha) <= 1e-13);
    CHECK(uot::max_abs_diff(fm.beta, ft.beta) <= 1e-13);
  }
  CHECK(mine == theirs);
  // Matrix<double>: the f64 kernel, as the reference template with T = double
  auto pd = uot::gen_problem_t<double>(30, 33, 50);
  uot::Matrix<double> md = pd.a, td = pd.a;
  uot::FusedState sd{uot::init_col_sums(md)}, tsd{uot::init_col_sums(td)};
  for (int it = 0; it < 3; ++it) {
    uot::cuda::fused_iterate(md, sd, pd, 0.6);
    uot::fused_iterate(td, tsd, pd, 0.6);
  }
  double m = 0.0;
  for (std::size_t k = 0; k < md.size(); ++k) m = std::max(m, std::abs(md.data()[k] - td.data()[k]) / td.data()[k]);
  CHECK(m <= 1e-13);
}

}  // namespace

int main() {
  const std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"solve matches the reference", test_solve_matches_reference},
      {"hand-checked iteration", test_hand_checked_iteration},
      {"per-iteration API", test_per_iteration_api_tracks_reference},
      {"session resumable + converges", test_session_is_resumable_and_converges},
      {"errors", test_errors_map_to_reference_exceptions},
      {"single-rank distributed", test_single_rank_distributed},
      {"ablation solvers", test_ablation_solvers_match_reference},
      {"problem files", test_problem_files_round_trip},
      {"single-rank peer distributed", test_single_rank_peer_distributed},
      {"Problem<double>", test_f64_problem_matches_reference},
      {"in-process ranks (reference signature)", test_in_process_ranks_match_reference},
      {"WorkerPlan overloads", test_worker_plan_overloads},
      {"integral 4th argument = workers", test_integral_fourth_argument_means_workers},
      {"fused_iterate inputs as given", test_fused_iterate_takes_inputs_as_given},
  };
  for (const auto& [name, fn] : cases) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "%s: unexpected exception: %s\n", name, e.what());
    }
    std::printf("%-34s %s\n", name, g_fail == before ? "PASS" : "FAIL");
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail;
}
