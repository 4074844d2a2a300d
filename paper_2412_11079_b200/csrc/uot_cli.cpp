// uot-cuda — the reference CLI's `gen`, `solve` and `bench` subcommands
// (tools/uot_main.cpp:184-364) with the B200 backend behind them, built only on
// the C ABI (include/uot_cuda.h). Same options, same JSON report keys
// (report_json, uot_main.cpp:118-130), same CSV header (uot_main.cpp:340), same
// exit codes (0 converged, 2 not converged, 1 error). Solvers: `cuda` (the
// fused sweep; `fused` and `parallel` are accepted as aliases), the GPU
// ablations `baseline` (baseline.hpp) and `tiled` (tiled.hpp two-pass), and
// `dist --ranks P` (uot_main.cpp:109-111, distributed_solve): P row-sharded
// ranks in this process over the visible GPUs (uot_create_group). `verify`
// (uot_main.cpp:131-175) runs them all and compares the plans with baseline's.
#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/uot_cuda.h"

namespace {

struct Args {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string str(const std::string& k, const std::string& d) const { return has(k) ? kv.at(k) : d; }
  uint64_t u64(const std::string& k, uint64_t d) const { return has(k) ? std::strtoull(kv.at(k).c_str(), nullptr, 10) : d; }
  double f64(const std::string& k, double d) const { return has(k) ? std::strtod(kv.at(k).c_str(), nullptr) : d; }
};

struct Fail {
  int code;
  std::string msg;
};

void check(uot_ctx* ctx, int rc) {
  if (rc != UOT_OK) throw Fail{rc, ctx ? uot_last_error(ctx) : "error"};
}

int parse_dtype(const std::string& s) {
  if (s == "fp32") return UOT_F32;
  if (s == "fp64") return UOT_F64;
  throw Fail{UOT_INVALID_PARAMETER, "dtype must be fp32 or fp64"};
}
const char* dtype_name(int d) { return d == UOT_F64 ? "fp64" : "fp32"; }

void emit(const std::string& text, const std::string& out) {
  if (out.empty()) {
    std::fputs(text.c_str(), stdout);
    return;
  }
  FILE* f = std::fopen(out.c_str(), "w");
  if (!f) throw Fail{UOT_IO_ERROR, "cannot open output file " + out};
  std::fputs(text.c_str(), f);
  std::fclose(f);
}

std::string num(double v) {  // JSON number, round-trippable
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// A session holding the problem of --in, or gen_problem(seed, m, n, dtype)
// generated in HBM (uot_main.cpp:52-62: er = ep = 1 for generated problems).
struct Loaded {
  uot_ctx* ctx = nullptr;
  uint64_t m = 0, n = 0;
  int dtype = UOT_F32;
  ~Loaded() { uot_destroy(ctx); }
};

void load(const Args& a, Loaded& L, int device) {
  if (a.has("in")) {
    const std::string path = a.kv.at("in");
    double er = 0, ep = 0;
    const int rc = uot_problem_file_info(path.c_str(), &L.m, &L.n, &L.dtype, &er, &ep);
    if (rc) throw Fail{rc, uot_last_io_error()};
    check(L.ctx, uot_create(&L.ctx, L.m, L.n, L.dtype, device));
    check(L.ctx, uot_load_problem_file(L.ctx, path.c_str()));
  } else {
    L.m = a.u64("m", 64);
    L.n = a.u64("n", 64);
    L.dtype = parse_dtype(a.str("dtype", "fp64"));
    check(L.ctx, uot_create(&L.ctx, L.m, L.n, L.dtype, device));
    check(L.ctx, uot_generate_problem(L.ctx, a.u64("seed", 1), 1.0, 1.0));
  }
}

int variant_of(const std::string& solver) {
  if (solver == "cuda" || solver == "fused" || solver == "parallel") return UOT_VARIANT_FUSED;
  if (solver == "baseline") return UOT_VARIANT_BASELINE;
  if (solver == "tiled") return UOT_VARIANT_TWO_PASS;
  throw Fail{UOT_INVALID_PARAMETER, "unknown solver '" + solver + "' (cuda|baseline|tiled)"};
}

struct Report {
  std::string solver;
  uint64_t iterations = 0;
  double final_error = 0.0, wall_ms = 0.0, device_ms = 0.0;
  bool converged = false;
};

Report run(uot_ctx* ctx, const std::string& solver, double tol, uint64_t max_iter) {
  const int v = variant_of(solver);
  if (!(tol > 0.0)) throw Fail{UOT_INVALID_PARAMETER, "tol must be positive"};
  if (max_iter < 1) throw Fail{UOT_INVALID_PARAMETER, "max_iter must be at least 1"};
  const auto t0 = std::chrono::steady_clock::now();
  check(ctx, uot_set_variant(ctx, v));
  check(ctx, uot_init_col_sums(ctx));
  Report r;
  int conv = 0;
  check(ctx, uot_iterate_timed(ctx, max_iter, tol, &r.iterations, &r.final_error, &conv, &r.device_ms));
  r.converged = conv != 0;
  r.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  r.solver = v == UOT_VARIANT_FUSED ? "cuda" : solver;
  return r;
}

// --solver dist: distributed_solve(p, tol, max_iter, ranks) (uot_main.cpp:109-111)
// as an in-process session group, rank r on --devices[r] (default: round robin).
struct Group {
  std::vector<uot_ctx*> ctx;
  ~Group() {
    for (auto* c : ctx) uot_destroy(c);
  }
  void check(int rc) const {
    if (rc == UOT_OK) return;
    std::string msg = "session group";
    for (auto* c : ctx)
      if (c && *uot_last_error(c)) msg = uot_last_error(c);
    throw Fail{rc, msg};
  }
};

Report run_dist(const Args& a, Group& g, uint64_t& m, uint64_t& n, int& dtype, double tol, uint64_t max_iter) {
  if (!(tol > 0.0)) throw Fail{UOT_INVALID_PARAMETER, "tol must be positive"};
  if (max_iter < 1) throw Fail{UOT_INVALID_PARAMETER, "max_iter must be at least 1"};
  const uint64_t ranks = a.u64("ranks", 2);  // uot_main.cpp:216 default
  if (ranks < 1 || ranks > 4096) throw Fail{UOT_PARTITION_ERROR, "RankPartition: ranks must be in [1, 4096]"};
  std::string path;
  if (a.has("in")) {
    path = a.kv.at("in");
    double er = 0, ep = 0;
    const int rc = uot_problem_file_info(path.c_str(), &m, &n, &dtype, &er, &ep);
    if (rc) throw Fail{rc, uot_last_io_error()};
  } else {
    m = a.u64("m", 64);
    n = a.u64("n", 64);
    dtype = parse_dtype(a.str("dtype", "fp64"));
  }
  std::vector<int> dev;
  if (a.has("devices")) {
    std::stringstream ss(a.kv.at("devices"));
    std::string t;
    while (std::getline(ss, t, ',')) dev.push_back(std::atoi(t.c_str()));
    if (dev.size() != ranks) throw Fail{UOT_INVALID_PARAMETER, "--devices needs one device per rank"};
  }
  g.ctx.assign(ranks, nullptr);
  g.check(uot_create_group(g.ctx.data(), m, n, dtype, dev.empty() ? nullptr : dev.data(), static_cast<int>(ranks),
                           nullptr));
  for (auto* c : g.ctx)  // each rank streams / generates only its row block
    g.check(path.empty() ? uot_generate_problem(c, a.u64("seed", 1), 1.0, 1.0) : uot_load_problem_file(c, path.c_str()));
  const auto t0 = std::chrono::steady_clock::now();
  g.check(uot_group_init_col_sums(g.ctx.data(), static_cast<int>(ranks)));
  Report r;
  int conv = 0;
  g.check(uot_group_iterate(g.ctx.data(), static_cast<int>(ranks), max_iter, tol, &r.iterations, &r.final_error, &conv));
  r.converged = conv != 0;
  r.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  r.solver = "dist";
  return r;
}

// The plan of a session (its rows) as doubles.
void plan_into(uot_ctx* ctx, int dtype, uint64_t rows, uint64_t n, double* out) {
  if (dtype == UOT_F64) {
    check(ctx, uot_get_plan_f64(ctx, out));
    return;
  }
  std::vector<float> f(rows * n);
  check(ctx, uot_get_plan(ctx, f.data()));
  for (size_t k = 0; k < f.size(); ++k) out[k] = f[k];
}

double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {  // matrix.hpp:66-73
  double m = 0.0;
  for (size_t k = 0; k < a.size(); ++k) m = std::max(m, std::fabs(a[k] - b[k]));
  return m;
}

// verify (uot_main.cpp:131-175): every solver for a fixed iteration count on
// the same problem, plans compared with the baseline's.
std::string verify(const Args& a, int device, bool& ok) {
  const uint64_t iters = a.u64("iters", 25), workers = a.u64("workers", 4), ranks = a.u64("ranks", 3);
  const double tol = a.f64("tol", 1e-10);
  std::map<std::string, std::vector<double>> plans;
  uint64_t m = 0, n = 0;
  int dt = UOT_F64;
  for (const char* solver : {"baseline", "fused", "parallel", "tiled"}) {
    Loaded L;
    load(a, L, device);
    m = L.m, n = L.n, dt = L.dtype;
    run(L.ctx, solver, 1e-300, iters);
    std::vector<double> p(m * n);
    plan_into(L.ctx, dt, m, n, p.data());
    plans[solver] = std::move(p);
  }
  const uint64_t eff_ranks = std::min<uint64_t>(ranks, m);
  {
    Args b = a;
    b.kv["ranks"] = std::to_string(eff_ranks);
    b.kv.erase("devices");
    Group g;
    uint64_t mm = 0, nn = 0;
    int dd = 0;
    run_dist(b, g, mm, nn, dd, 1e-300, iters);
    std::vector<double> p(m * n);
    for (auto* c : g.ctx) {
      uot_layout l{};
      g.check(uot_get_layout(c, &l));
      plan_into(c, dt, l.rows, n, p.data() + l.row_offset * n);
    }
    plans["dist"] = std::move(p);
  }
  const auto& base = plans["baseline"];
  const double d_fused = max_abs_diff(base, plans["fused"]), d_par = max_abs_diff(base, plans["parallel"]),
               d_tiled = max_abs_diff(base, plans["tiled"]), d_dist = max_abs_diff(base, plans["dist"]);
  const double d_max = std::max({d_fused, d_par, d_tiled, d_dist});
  ok = d_max <= tol;
  std::ostringstream js;
  js << "{\n  \"iterations\": " << iters << ",\n  \"workers\": " << workers << ",\n  \"ranks\": " << eff_ranks
     << ",\n  \"diff_vs_baseline\": {\n    \"fused\": " << num(d_fused) << ",\n    \"parallel\": " << num(d_par)
     << ",\n    \"tiled\": " << num(d_tiled) << ",\n    \"dist\": " << num(d_dist) << "\n  },\n  \"max_diff\": "
     << num(d_max) << ",\n  \"tolerance\": " << num(tol) << ",\n  \"ok\": " << (ok ? "true" : "false") << "\n}\n";
  return js.str();
}

// write_problem's container (problem_io.cpp:97-104) straight from the host generator.
void write_generated(const std::string& path, uint64_t seed, uint64_t m, uint64_t n, int dtype) {
  const size_t es = dtype == UOT_F64 ? 8 : 4;
  std::vector<unsigned char> a(m * n * es);
  std::vector<double> rpd(m), cpd(n);
  const int rc = dtype == UOT_F64
                     ? uot_gen_block_f64(seed, m, n, 0, m, reinterpret_cast<double*>(a.data()), rpd.data(), cpd.data(), 64)
                     : uot_gen_block_f32(seed, m, n, 0, m, reinterpret_cast<float*>(a.data()), rpd.data(), cpd.data(), 64);
  if (rc) throw Fail{rc, "gen: matrix must be at least 1x1"};
  unsigned char h[40] = {'U', 'O', 'T', 'P', 1, 0, static_cast<unsigned char>(dtype), 0};
  for (int k = 0; k < 8; ++k) h[8 + k] = static_cast<unsigned char>(m >> (8 * k));
  for (int k = 0; k < 8; ++k) h[16 + k] = static_cast<unsigned char>(n >> (8 * k));
  const double one = 1.0;
  std::memcpy(h + 24, &one, 8);
  std::memcpy(h + 32, &one, 8);
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw Fail{UOT_IO_ERROR, "write_problem: cannot open " + path};
  const bool ok = std::fwrite(h, 1, 40, f) == 40 && std::fwrite(a.data(), 1, a.size(), f) == a.size() &&
                  std::fwrite(rpd.data(), 8, m, f) == m && std::fwrite(cpd.data(), 8, n, f) == n;
  std::fclose(f);
  if (!ok) throw Fail{UOT_IO_ERROR, "write_problem: short write to " + path};
}

void usage() {
  std::puts(
      "uot-cuda: the reference CLI (tools/uot_main.cpp) on a B200\n"
      "  gen   --out FILE [--seed S] [--m M] [--n N] [--dtype fp32|fp64]\n"
      "  solve [--in FILE | --seed S --m M --n N --dtype fp32|fp64] [--solver cuda|baseline|tiled|dist]\n"
      "        [--tol T] [--max-iter K] [--out REPORT.json] [--plan-out FILE] [--device D]\n"
      "        [--ranks P [--devices 0,1,..]]   (dist: P row-sharded ranks over the GPUs)\n"
      "  verify [--in FILE | --seed S --m M --n N --dtype fp32|fp64] [--iters 25] [--workers 4] [--ranks 3]\n"
      "        [--tol 1e-10] [--out REPORT.json] [--device D]   (every solver vs baseline: exit 0 ok, 2 not)\n"
      "  bench [--sizes 256,512,1024] [--solvers cuda,baseline] [--iters K] [--seed S] [--dtype fp32|fp64]\n"
      "        [--out FILE.csv] [--device D]\n"
      "exit: 0 ok / converged, 2 not converged, 1 error");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
    usage();
    return argc < 2 ? 1 : 0;
  }
  const std::string cmd = argv[1];
  Args a;
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0 || i + 1 >= argc) {
      std::fprintf(stderr, "error: expected --option value, got '%s'\n", argv[i]);
      return 1;
    }
    a.kv[k.substr(2)] = argv[++i];
  }
  const int device = static_cast<int>(a.u64("device", 0));
  try {
    if (cmd == "gen") {
      if (!a.has("out")) throw Fail{UOT_INVALID_PARAMETER, "gen: --out is required"};
      write_generated(a.kv.at("out"), a.u64("seed", 1), a.u64("m", 64), a.u64("n", 64),
                      parse_dtype(a.str("dtype", "fp64")));
      return 0;
    }
    if (cmd == "solve" && a.str("solver", "cuda") == "dist") {
      Group g;
      uint64_t m = 0, n = 0;
      int dt = UOT_F32;
      const Report r = run_dist(a, g, m, n, dt, a.f64("tol", 1e-6), a.u64("max-iter", 10000));
      if (a.has("plan-out"))
        for (auto* c : g.ctx) g.check(uot_save_problem_file(c, a.kv.at("plan-out").c_str()));
      std::ostringstream js;  // report_json (uot_main.cpp:118-130)
      js << "{\n  \"solver\": \"dist\",\n  \"M\": " << m << ",\n  \"N\": " << n << ",\n  \"dtype\": \""
         << dtype_name(dt) << "\",\n  \"workers\": 1,\n  \"ranks\": " << g.ctx.size() << ",\n"
         << "  \"iterations\": " << r.iterations << ",\n  \"final_error\": " << num(r.final_error)
         << ",\n  \"converged\": " << (r.converged ? "true" : "false") << ",\n  \"wall_ms\": " << num(r.wall_ms)
         << "\n}\n";
      emit(js.str(), a.str("out", ""));
      return r.converged ? 0 : 2;
    }
    if (cmd == "solve") {
      Loaded L;
      load(a, L, device);
      const Report r = run(L.ctx, a.str("solver", "cuda"), a.f64("tol", 1e-6), a.u64("max-iter", 10000));
      if (a.has("plan-out")) check(L.ctx, uot_save_problem_file(L.ctx, a.kv.at("plan-out").c_str()));
      std::ostringstream js;  // report_json (uot_main.cpp:118-130) + the device time
      js << "{\n  \"solver\": \"" << r.solver << "\",\n  \"M\": " << L.m << ",\n  \"N\": " << L.n
         << ",\n  \"dtype\": \"" << dtype_name(L.dtype) << "\",\n  \"workers\": 1,\n  \"ranks\": 1,\n"
         << "  \"iterations\": " << r.iterations << ",\n  \"final_error\": " << num(r.final_error)
         << ",\n  \"converged\": " << (r.converged ? "true" : "false") << ",\n  \"wall_ms\": " << num(r.wall_ms)
         << ",\n  \"device_ms\": " << num(r.device_ms) << "\n}\n";
      emit(js.str(), a.str("out", ""));
      return r.converged ? 0 : 2;
    }
    if (cmd == "verify") {
      bool ok = false;
      emit(verify(a, device, ok), a.str("out", ""));
      return ok ? 0 : 2;
    }
    if (cmd == "bench") {
      std::vector<uint64_t> sizes;
      std::vector<std::string> solvers;
      {
        std::stringstream ss(a.str("sizes", "256,512,1024"));
        std::string t;
        while (std::getline(ss, t, ',')) sizes.push_back(std::strtoull(t.c_str(), nullptr, 10));
        std::stringstream s2(a.str("solvers", "cuda,baseline"));
        while (std::getline(s2, t, ',')) solvers.push_back(t);
      }
      const int dt = parse_dtype(a.str("dtype", "fp32"));
      const uint64_t iters = a.u64("iters", 10);
      std::ostringstream csv;
      csv << "M,N,solver,workers,iterations,wall_ms,bytes_modeled\n";  // uot_main.cpp:340
      for (const uint64_t size : sizes) {
        for (const std::string& solver : solvers) {
          Loaded L;
          L.m = L.n = size;
          L.dtype = dt;
          check(L.ctx, uot_create(&L.ctx, size, size, dt, device));
          check(L.ctx, uot_generate_problem(L.ctx, a.u64("seed", 1), 1.0, 1.0));
          const Report r = run(L.ctx, solver, 1e-300, iters);
          // traffic_model (metrics.cpp:60-77): baseline 6 accesses per element, fused 2
          const uint64_t es = dt == UOT_F64 ? 8 : 4;
          const uint64_t bytes = (variant_of(solver) == UOT_VARIANT_BASELINE ? 6 : 2) * size * size * es * r.iterations;
          char ms[64];
          std::snprintf(ms, sizeof ms, "%.6g", r.device_ms);
          csv << size << ',' << size << ',' << r.solver << ",1," << r.iterations << ',' << ms << ',' << bytes << '\n';
        }
      }
      emit(csv.str(), a.str("out", ""));
      return 0;
    }
    usage();
    return 1;
  } catch (const Fail& f) {
    std::fprintf(stderr, "error: %s\n", f.msg.c_str());
    return 1;
  }
}
