// uot_cuda.cu — host runtime of the B200-native fused Sinkhorn-UOT path and its
// C ABI (include/uot_cuda.h). One session = one problem resident in HBM on one
// GPU (or one rank's row block of it), driven on one CUDA stream.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/uot_cuda.h"
#include "finalize.cuh"
#include "problem.cuh"
#include "sweep.cuh"
#include "resident.cuh"
#include "ablation.cuh"

using namespace uotk;

namespace {

constexpr unsigned kSliceMax = 8192;      // floats of a row one CTA owns when G == 1 (32 KiB)
constexpr unsigned kSliceMaxXchg = 8192;  // ... when a row spans G > 1 CTAs

// ------------------------------------------------------------ kernel table --
using SweepFn = void (*)(const SweepArgs);
struct SweepCfg {
  int nt, v, bm, nbuf, nf;
  bool xchg;           // rows span G > 1 CTAs (cross-CTA row-sum exchange)
  SweepFn iter[2];     // [FULL] iteration kernel
  SweepFn seed[2];     // [FULL] init_col_sums kernel
  size_t (*smem_bytes)(unsigned buf_stride);
};

// Sweep 2 lags sweep 1 by kLag = 2 extra batches (the factor warps' budget: the
// pow and, for G > 1, the L2 exchange round trip). Factor warps alternate
// batches: 3 (with split sweep roles the factor chain of a G > 1 group — warp
// partials, L2 exchange, f64 pow — paces sweep 2: 3 warps measured -1.5% at
// 32768^2 against 2; 4 warps exceed the register budget. Before the split, 2
// were faster for G > 1: more warps polling L2 cost more issue slots.)
// (Measured: a lag of 3 for G > 1 — more slack between a group's CTAs — is
// 10-15% slower: the 7-slot ring then prefetches only two batches.)
// L2 bytes (all CTAs together) written evict_last at the end of a streaming sweep
// and read first by the next one (measured 48, 64, 88 MiB: 48 MiB best at 8192^2,
// -3% per iteration; +-0 at the HBM-sized configs; the 126 MB L2 also holds the
// column partials and the stream's own lines).
constexpr uint64_t kKeepL2Bytes = 48ull << 20;
constexpr int kLag = 2;
constexpr int kLagX = 2;
constexpr int kFactorWarpsG1 = 3;
constexpr int kFactorWarpsX = 3;
// Column factors of sweep 1 parked in TMEM (sweep.cuh, TB) for slices of 3-4
// float4 per thread: frees the registers that otherwise spill (measured +5-8%
// at 32768^2 .. 16384^2; at V = 2 the factors fit registers and TMEM loses).
template <int NT, int V, int BM, int NB, bool XCHG = false>
SweepCfg make_cfg() {
  constexpr int NF = XCHG ? kFactorWarpsX : kFactorWarpsG1;
  SweepCfg c{};
  c.nt = NT;
  c.v = V;
  c.bm = BM;
  c.nbuf = NB;
  c.nf = NF;
  c.xchg = XCHG;
  constexpr bool TB = V >= 3;
  constexpr int LA = XCHG ? kLagX : kLag;
  c.iter[0] = sweep_kernel<NT, V, BM, NB, LA, XCHG, NF, false, false, float, TB>;
  c.iter[1] = sweep_kernel<NT, V, BM, NB, LA, XCHG, NF, true, false, float, TB>;
  c.seed[0] = sweep_kernel<NT, V, BM, NB, 1, false, 1, false, true>;
  c.seed[1] = sweep_kernel<NT, V, BM, NB, 1, false, 1, true, true>;
  c.smem_bytes = &SweepSmem<NT / 32, BM, NB>::bytes;
  return c;
}

// Resident (whole solve in one launch, matrix in shared memory) variants.
using ResidentFn = void (*)(const ResidentArgs);
struct ResidentCfg {
  int nt, v;
  ResidentFn fn[2];  // [FULL]
  size_t (*smem_bytes)(unsigned rows_cta, unsigned pitch);
};
template <int NT, int V>
ResidentCfg make_rcfg() {
  ResidentCfg c{};
  c.nt = NT;
  c.v = V;
  c.fn[0] = resident_kernel<NT, V, false>;
  c.fn[1] = resident_kernel<NT, V, true>;
  c.smem_bytes = &ResidentSmem<NT, V>::bytes;
  return c;
}
const std::vector<ResidentCfg>& rcfg_table() {
  static const std::vector<ResidentCfg> t = {make_rcfg<128, 1>(), make_rcfg<256, 1>(), make_rcfg<512, 1>(),
                                             make_rcfg<512, 2>(), make_rcfg<512, 4>()};
  return t;
}

// Problem<double>: the same kernel over fp64 storage (double2 chunks, 32 KiB =
// 4096-double slices); the ring/TMEM/persistent variants are fp32-only.
template <int NT, int V, int BM, int NB, bool XCHG = false>
SweepCfg make_cfg_f64() {
  constexpr int NF = XCHG ? kFactorWarpsX : kFactorWarpsG1;
  SweepCfg c{};
  c.nt = NT;
  c.v = V;
  c.bm = BM;
  c.nbuf = NB;
  c.nf = NF;
  c.xchg = XCHG;
  constexpr int LA = XCHG ? kLagX : kLag;
  c.iter[0] = sweep_kernel<NT, V, BM, NB, LA, XCHG, NF, false, false, double>;
  c.iter[1] = sweep_kernel<NT, V, BM, NB, LA, XCHG, NF, true, false, double>;
  c.seed[0] = sweep_kernel<NT, V, BM, NB, 1, false, 1, false, true, double>;
  c.seed[1] = sweep_kernel<NT, V, BM, NB, 1, false, 1, true, true, double>;
  c.smem_bytes = &SweepSmem<NT / 32, BM, NB>::bytes;
  return c;
}
const std::vector<SweepCfg>& cfg_table_f64() {
  static const std::vector<SweepCfg> t = {
      make_cfg_f64<128, 1, 4, 7>(), make_cfg_f64<256, 1, 8, 7>(), make_cfg_f64<512, 1, 4, 7>(),
      make_cfg_f64<512, 2, 2, 7>(), make_cfg_f64<512, 4, 1, 7>(),
      make_cfg_f64<512, 3, 1, 7, true>(), make_cfg_f64<512, 4, 1, 7, true>(),
  };
  return t;
}

const std::vector<SweepCfg>& cfg_table() {
  static const std::vector<SweepCfg> t = {
      // G == 1 (rows fit one CTA): 32 KiB ring slots
      make_cfg<128, 1, 4, 7>(), make_cfg<256, 1, 8, 7>(), make_cfg<512, 1, 4, 7>(),
      make_cfg<512, 2, 2, 7>(), make_cfg<512, 3, 1, 7>(), make_cfg<512, 4, 1, 7>(),
      // G > 1: 32 KiB slices; two factor warps overlap the exchange round trips
      make_cfg<512, 3, 1, 7, true>(), make_cfg<512, 4, 1, 7, true>(),
  };
  return t;
}

// ------------------------------------------------------------------- NCCL --
// Loaded on first multi-GPU use so single-GPU sessions never touch libnccl.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string err;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.CommDestroy && a.GetErrorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

unsigned round_up(unsigned x, unsigned m) { return (x + m - 1) / m * m; }

__global__ void smid_probe_kernel(unsigned* out) {
  extern __shared__ unsigned char probe_smem[];
  if (threadIdx.x == 0) {
    probe_smem[0] = 0;
    out[blockIdx.x] = uotk::smid();
  }
}

void balanced_bounds(uint64_t k, uint64_t rows, uint64_t* bounds) {  // plan.cpp:11-21
  const uint64_t base = rows / k, rem = rows % k;
  bounds[0] = 0;
  for (uint64_t w = 0; w < k; ++w) bounds[w + 1] = bounds[w] + base + (w < rem ? 1 : 0);
}

struct Status {
  int code;
  std::string msg;
};

}  // namespace

struct uot_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sms = 0;
  uint64_t rows = 0, cols = 0, row_offset = 0, global_rows = 0;
  int rank = 0, nranks = 1;
  bool is_dist = false;  // created by uot_create_dist / uot_create_peer (CommStats are kept)
  int xmode = kXchNone;  // how the column sums of the ranks are combined
  ncclComm_t comm = nullptr;
  // kXchPeer: this rank's exchange region, every rank's region mapped here
  unsigned char* region = nullptr;
  size_t region_bytes = 0;
  unsigned xlen = 0;
  std::vector<unsigned char*> peer_ptrs;  // [nranks]; own entry = region
  unsigned char** d_peers = nullptr;      // device copy of peer_ptrs
  bool connected = false;
  bool group_local = false;  // a rank of a single-process group (uot_create_group): direct peer pointers, no IPC
  uint64_t group_id = 0;     // which uot_create_group call made this rank (collectives check it)
  cudaEvent_t xev = nullptr;  // group: stage 1 of the running exchange is enqueued (cross-rank stream order)

  // layout
  unsigned G = 1, slice = 0, pitch = 0, groups = 1, B = 1, buf_stride = 0, grid = 1;
  size_t smem = 0;
  const SweepCfg* cfg = nullptr;
  int evict_first = 0;
  unsigned keep = 0;  // batches per CTA stored L2-resident for the next sweep (SweepArgs::keep)
  int full = 0;
  int smid_map = 0;
  int dyn = 1;  // batches handed out by a global counter (SweepArgs::dyn)
  int schedule = UOT_SCHEDULE_UNIFORM;  // uot_set_schedule
  bool pinned = false;              // one sweep CTA on every SM: CTA slot = %smid (d_slot)
  unsigned* d_slot = nullptr;       // [sms] CTA slot of each SM (identity)
  unsigned long long* d_gbounds = nullptr;  // [groups+1] weighted static row blocks (UOT_SCHEDULE_WEIGHTED)
  unsigned* d_dbg = nullptr;        // [grid][kDbg] {smid, batches, start, end} of the last sweep
  std::vector<uint32_t> weights;    // per row group (UOT_SCHEDULE_WEIGHTED)
  ulonglong2* mail = nullptr;  // [groups][kMail] batch picks of the group leaders
  // resident mode: the whole uot_iterate call is one persistent launch
  const ResidentCfg* rcfg = nullptr;
  unsigned rgrid = 0;
  size_t rsmem = 0;
  int rfull = 0;
  bool resident_on = true;  // uot_set_resident: use rcfg when the problem fits
  bool wide = false;  // rows wider than #SMs slices: only the two-pass schedule (ablation.cuh) runs

  // device buffers
  void* P = nullptr;          // [rows][pitch] of `dtype` (float or double)
  int dtype = UOT_F32;
  unsigned esz = 4;           // bytes per element
  float* Pf() const { return static_cast<float*>(P); }
  double *rpd = nullptr, *cpd = nullptr, *alpha = nullptr, *beta2 = nullptr, *col_sums = nullptr,
         *xsum = nullptr, *partials = nullptr, *cta_err = nullptr;
  ulonglong2* xrec = nullptr;
  Control* ctl = nullptr;
  int* dflag = nullptr;
  unsigned* bar_flags = nullptr;  // resident kernel's grid barrier (one epoch per CTA)
  // iteration schedule (uot_set_variant): fused sweep, or the two ablations
  int variant = UOT_VARIANT_FUSED;
  double *abl_partials = nullptr, *abl_row_err = nullptr;
  unsigned abl_gx = 0, abl_gy = 0, abl_rowctas = 0;
  Control* h_ctl = nullptr;  // pinned mirror

  double fi = 0.0;
  double er = 1.0, ep = 1.0;  // the Problem's coefficients (written back by uot_save_problem_file)
  bool have_problem = false, seeded = false;

  bool timing = false;
  std::vector<cudaEvent_t> ev;
  double sweep_ms = 0.0, fin_ms = 0.0;
  uint64_t sweeps_timed = 0;
  uint64_t launches = 0;

  std::string last_error;

  int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    last_error = buf;
    return code;
  }
  int cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return UOT_OK;
    return fail(UOT_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
  }
};

#define CK(expr)                                              \
  do {                                                        \
    const int _rc = ctx->cuda((expr), #expr);                 \
    if (_rc != UOT_OK) return _rc;                            \
  } while (0)

namespace {

// G > 1 and one sweep CTA on every SM: address CTAs by %smid so the G CTAs of a
// row group run on neighbouring SMs. Enabled only when a probe launch with the
// sweep's footprint shows %smid is a permutation of [0, grid).
int probe_smid_map(uot_ctx* ctx) {
  ctx->smid_map = 0;
  int nsm = 0;
  if (ctx->cuda(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device), "attr")) return UOT_CUDA_ERROR;
  if (ctx->G < 2 || static_cast<int>(ctx->grid) != nsm) return UOT_OK;
  unsigned* d = nullptr;
  CK(cudaMalloc(&d, ctx->grid * sizeof(unsigned)));
  CK(cudaFuncSetAttribute(smid_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ctx->smem)));
  smid_probe_kernel<<<ctx->grid, 32, ctx->smem, ctx->stream>>>(d);
  std::vector<unsigned> h(ctx->grid);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d, ctx->grid * sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d);
  CK(e);
  std::vector<char> seen(ctx->grid, 0);
  for (unsigned v : h) {
    if (v >= ctx->grid || seen[v]) return UOT_OK;
    seen[v] = 1;
  }
  ctx->smid_map = 1;
  return UOT_OK;
}

// One sweep CTA on every SM (the grid covers the SMs and two CTAs cannot share
// one): CTA slots are pinned to SMs (slot = %smid), so a row group is the same
// physical SMs in every launch and a static weighted row split
// (UOT_SCHEDULE_WEIGHTED) stays attached to the SMs it was measured on.
void plan_pinning(uot_ctx* ctx, int smem_optin) {
  ctx->pinned = ctx->grid == static_cast<unsigned>(ctx->sms) &&
                2 * ctx->smem > static_cast<size_t>(smem_optin) + 1024;
}

// Row bounds of the groups from integer weights: group g owns
// [rows * W(g) / W, rows * W(g+1) / W) with W(g) the prefix sum.
std::vector<unsigned long long> weighted_bounds(uint64_t rows, const std::vector<uint32_t>& w) {
  uint64_t wsum = 0;
  for (uint32_t x : w) wsum += x;
  std::vector<unsigned long long> b(w.size() + 1, 0);
  uint64_t acc = 0;
  for (size_t g = 0; g < w.size(); ++g) {
    acc += w[g];
    b[g + 1] = static_cast<unsigned long long>(static_cast<unsigned __int128>(rows) * acc / wsum);
  }
  return b;
}

int plan_layout(uot_ctx* ctx) {
  const uint64_t cols = ctx->cols;
  if (cols > (1ull << 26)) return ctx->fail(UOT_CONFIG_ERROR, "cols %llu too large", (unsigned long long)cols);
  const bool f64 = ctx->dtype == UOT_F64;
  const unsigned epc = 16 / ctx->esz;  // elements per 16-byte chunk
  const unsigned smax = kSliceMax * 4 / ctx->esz;  // 32 KiB of elements
  const unsigned xmax = kSliceMaxXchg * 4 / ctx->esz;
  unsigned G = cols <= smax ? 1u : static_cast<unsigned>((cols + xmax - 1) / xmax);
  if (G > static_cast<unsigned>(ctx->sms)) {
    // Rows wider than one slice per SM: the fused sweep cannot hold a row across
    // the grid, so a single-rank session runs the paper's two-pass schedule
    // (ablation.cuh: warp-per-row and column kernels, any width, the same
    // arithmetic at 16 B per element) for the seed and every iteration.
    if (ctx->nranks > 1)
      return ctx->fail(UOT_CONFIG_ERROR, "cols %llu needs %u CTAs per row (max %d)",
                       (unsigned long long)cols, G, ctx->sms);
    ctx->wide = true;
    ctx->G = 1;
    ctx->slice = ctx->pitch = round_up(static_cast<unsigned>(cols), 4);
    ctx->cfg = &(f64 ? cfg_table_f64() : cfg_table()).front();  // (layout reporting only: no sweep launches)
    ctx->B = 1;
    ctx->groups = ctx->grid = 1;
    ctx->buf_stride = 128;
    ctx->dyn = 0;
    return UOT_OK;
  }
  const unsigned slice = round_up(static_cast<unsigned>((cols + G - 1) / G), epc);
  const SweepCfg* cfg = nullptr;
  for (const auto& c : f64 ? cfg_table_f64() : cfg_table())
    if (static_cast<unsigned>(c.nt) * epc * c.v >= slice && c.xchg == (G > 1)) {
      cfg = &c;
      break;
    }
  if (!cfg) return ctx->fail(UOT_CONFIG_ERROR, "no sweep configuration covers a %u-element slice", slice);
  ctx->G = G;
  ctx->slice = slice;
  ctx->pitch = slice * G;
  ctx->cfg = cfg;
  ctx->B = G > 1 ? 1u : std::max(1u, std::min(static_cast<unsigned>(cfg->bm), smax / slice));
  ctx->groups = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(ctx->rows, ctx->sms / G)));
  ctx->grid = ctx->groups * G;
  ctx->buf_stride = round_up(ctx->B * slice * ctx->esz, 128);
  ctx->smem = cfg->smem_bytes(ctx->buf_stride);
  int smem_optin = 0;
  CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  ctx->evict_first = static_cast<uint64_t>(ctx->rows) * ctx->pitch * ctx->esz > (64ull << 20) ? 1 : 0;
  // Streaming problems keep the last kKeepL2Bytes of every CTA's sweep in L2 for
  // the next sweep, which walks the blocks the other way (SweepArgs::keep).
  ctx->keep = ctx->evict_first
                  ? static_cast<unsigned>(kKeepL2Bytes / (static_cast<uint64_t>(ctx->grid) * ctx->B * slice * ctx->esz))
                  : 0u;
  // Row-batch schedule: fixed row blocks (bit-reproducible run to run, as the
  // reference's ordered reduction) unless the caller opts into the dynamic
  // batch counter with uot_set_deterministic(ctx, 0).
  ctx->dyn = 0;
  ctx->full = slice == epc * cfg->nt * cfg->v ? 1 : 0;
  int rc = probe_smid_map(ctx);
  if (rc) return rc;
  plan_pinning(ctx, smem_optin);
  for (SweepFn fn : {cfg->iter[ctx->full], cfg->seed[ctx->full]}) {
    if (!fn) continue;
    const int rc = ctx->cuda(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(ctx->smem)),
                             "cudaFuncSetAttribute(smem)");
    if (rc) return rc;
  }
  // Resident mode (resident.cuh): one rank, rows fit one CTA (G == 1), a CTA's
  // row block fits shared memory and at most 32 rows per CTA (uot_set_resident).
  ctx->rcfg = nullptr;
  if (!f64 && ctx->nranks == 1 && G == 1) {
    const unsigned rgrid = static_cast<unsigned>(std::min<uint64_t>(ctx->rows, ctx->sms));
    const uint64_t rows_cta = (ctx->rows + rgrid - 1) / rgrid;
    const unsigned nq = ctx->pitch / 4;
    for (const auto& rc : rcfg_table()) {
      if (static_cast<unsigned>(rc.nt * rc.v) < nq) continue;
      const size_t sm = rc.smem_bytes(static_cast<unsigned>(rows_cta), ctx->pitch);
      if (rows_cta <= 32 && sm <= static_cast<size_t>(smem_optin)) {
        ctx->rcfg = &rc;
        ctx->rgrid = rgrid;
        ctx->rsmem = sm;
        ctx->rfull = nq == static_cast<unsigned>(rc.nt * rc.v) ? 1 : 0;
        CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(rc.fn[ctx->rfull]),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
      }
      break;
    }
  }
  return UOT_OK;
}

template <typename T>
int dalloc(uot_ctx* ctx, T** p, size_t count) {
  return ctx->cuda(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)),
                   "cudaMalloc");
}

int alloc_all(uot_ctx* ctx) {
  const size_t rows = ctx->rows, pitch = ctx->pitch;
  int rc;
  if ((rc = ctx->cuda(cudaMalloc(&ctx->P, std::max<size_t>(rows * pitch, 1) * ctx->esz), "cudaMalloc"))) return rc;
  if ((rc = dalloc(ctx, &ctx->rpd, rows))) return rc;
  if ((rc = dalloc(ctx, &ctx->alpha, rows))) return rc;
  if ((rc = dalloc(ctx, &ctx->cpd, pitch))) return rc;
  if ((rc = dalloc(ctx, &ctx->beta2, 2 * pitch))) return rc;
  if ((rc = dalloc(ctx, &ctx->col_sums, pitch))) return rc;
  if ((rc = dalloc(ctx, &ctx->xsum, pitch + ctx->nranks))) return rc;
  if ((rc = dalloc(ctx, &ctx->partials, static_cast<size_t>(ctx->groups) * pitch))) return rc;
  if ((rc = dalloc(ctx, &ctx->cta_err, kErrSlots * static_cast<size_t>(ctx->grid)))) return rc;
  const size_t xn = static_cast<size_t>(ctx->grid) * kRing;
  if ((rc = dalloc(ctx, &ctx->xrec, xn))) return rc;
  const size_t mn = static_cast<size_t>(ctx->grid) * kMail;  // >= groups * kMail
  if ((rc = dalloc(ctx, &ctx->mail, mn))) return rc;
  if ((rc = dalloc(ctx, &ctx->d_dbg, kDbg * static_cast<size_t>(ctx->grid)))) return rc;
  CK(cudaMemsetAsync(ctx->d_dbg, 0, kDbg * sizeof(unsigned) * ctx->grid, ctx->stream));
  if (ctx->pinned) {
    std::vector<unsigned> slot(ctx->sms);
    for (int i = 0; i < ctx->sms; ++i) slot[i] = static_cast<unsigned>(i);
    if ((rc = dalloc(ctx, &ctx->d_slot, slot.size()))) return rc;
    if ((rc = dalloc(ctx, &ctx->d_gbounds, static_cast<size_t>(ctx->groups) + 1))) return rc;
    CK(cudaMemcpy(ctx->d_slot, slot.data(), sizeof(unsigned) * slot.size(), cudaMemcpyHostToDevice));
  }
  CK(cudaMemsetAsync(ctx->mail, 0, mn * sizeof(ulonglong2), ctx->stream));
  if ((rc = dalloc(ctx, &ctx->ctl, 1))) return rc;
  if ((rc = dalloc(ctx, &ctx->dflag, 1))) return rc;
  if ((rc = dalloc(ctx, &ctx->bar_flags, std::max<size_t>(ctx->grid, ctx->sms)))) return rc;
  CK(cudaMemsetAsync(ctx->bar_flags, 0, std::max<size_t>(ctx->grid, ctx->sms) * sizeof(unsigned), ctx->stream));
  if ((rc = ctx->cuda(cudaMallocHost(&ctx->h_ctl, sizeof(Control)), "cudaMallocHost"))) return rc;
  CK(cudaMemsetAsync(ctx->xrec, 0, xn * sizeof(ulonglong2), ctx->stream));
  CK(cudaMemsetAsync(ctx->ctl, 0, sizeof(Control), ctx->stream));
  CK(cudaMemsetAsync(ctx->beta2, 0, 2 * pitch * sizeof(double), ctx->stream));
  CK(cudaMemsetAsync(ctx->cpd, 0, pitch * sizeof(double), ctx->stream));
  return UOT_OK;
}

int create_common(uot_ctx* ctx, int device) {
  ctx->device = device;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return ctx->fail(UOT_INVALID_PARAMETER, "device %d out of range (%d visible)", device, ndev);
  CK(cudaSetDevice(device));
  CK(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device));
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  int rc = plan_layout(ctx);
  if (rc) return rc;
  if ((rc = alloc_all(ctx))) return rc;
  return ctx->wide ? uot_set_variant(ctx, UOT_VARIANT_TWO_PASS) : UOT_OK;
}

SweepArgs sweep_args(const uot_ctx* ctx) {
  SweepArgs a;
  a.P = ctx->P;
  a.beta2 = ctx->beta2;
  a.rpd = ctx->rpd;
  a.alpha = ctx->alpha;
  a.partials = ctx->partials;
  a.cta_err = ctx->cta_err;
  a.xrec = ctx->xrec;
  a.ctl = ctx->ctl;
  a.rows = ctx->rows;
  a.pitch = ctx->pitch;
  a.slice = ctx->slice;
  a.G = ctx->G;
  a.groups = ctx->groups;
  a.B = ctx->B;
  a.buf_stride = ctx->buf_stride;
  a.evict_first = ctx->evict_first;
  a.smid_map = ctx->smid_map;
  a.dyn = ctx->dyn;
  a.keep = ctx->keep;
  a.slot_of_sm = ctx->pinned ? ctx->d_slot : nullptr;
  a.gbounds = ctx->pinned && ctx->schedule == UOT_SCHEDULE_WEIGHTED ? ctx->d_gbounds : nullptr;
  a.dbg = ctx->d_dbg;
  a.mail = ctx->mail;
  a.fi = ctx->fi;
  return a;
}

FinalizeArgs fin_args(const uot_ctx* ctx) {
  FinalizeArgs f;
  f.partials = ctx->partials;
  f.cta_err = ctx->cta_err;
  f.cpd = ctx->cpd;
  f.beta2 = ctx->beta2;
  f.col_sums = ctx->col_sums;
  f.xsum = ctx->xsum;
  f.ctl = ctx->ctl;
  f.cols = static_cast<unsigned>(ctx->cols);
  f.pitch = ctx->pitch;
  f.groups = ctx->groups;
  f.grid = ctx->grid;
  f.rank = static_cast<unsigned>(ctx->rank);
  f.nranks = static_cast<unsigned>(ctx->nranks);
  f.peers = ctx->d_peers;
  f.region = ctx->region;
  f.xlen = ctx->xlen;
  f.fi = ctx->fi;
  return f;
}

int launch_sweep(uot_ctx* ctx, bool seed) {
  const SweepArgs a = sweep_args(ctx);
  // cooperative whenever G > 1: the iteration's CTAs spin on each other, and with
  // smid_map a CTA's identity is its SM — only a co-resident grid (one CTA per
  // SM) makes that a permutation, even for the seed sweep, when other kernels
  // share the GPU (e.g. the ranks of a session group on one device)
  const bool xchg = ctx->G > 1 || ctx->pinned;
  SweepFn fn = seed ? ctx->cfg->seed[ctx->full] : ctx->cfg->iter[ctx->full];
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(ctx->grid);
  // compute warps + producer warp + factor warp(s)
  lc.blockDim = dim3(ctx->cfg->nt + 32 * (1 + (seed ? 1 : ctx->cfg->nf)));
  lc.dynamicSmemBytes = ctx->smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // CTAs of a group spin on each other
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = xchg ? 1 : 0;
  ctx->launches++;
  return ctx->cuda(cudaLaunchKernelEx(&lc, fn, a), "sweep launch");
}

// ------------------------------------------------------------ ablations --
AblArgs abl_args(const uot_ctx* ctx) {
  AblArgs a;
  a.P = ctx->P;
  a.beta2 = ctx->beta2;
  a.rpd = ctx->rpd;
  a.alpha = ctx->alpha;
  a.partials = ctx->abl_partials;
  a.row_err = ctx->abl_row_err;
  a.ctl = ctx->ctl;
  a.rows = ctx->rows;
  a.cols = static_cast<unsigned>(ctx->cols);
  a.pitch = ctx->pitch;
  a.gy = ctx->abl_gy;
  a.fi = ctx->fi;
  return a;
}

FinalizeArgs abl_fin_args(const uot_ctx* ctx) {
  FinalizeArgs f = fin_args(ctx);
  f.partials = ctx->abl_partials;
  f.groups = ctx->abl_gy;
  f.cta_err = ctx->abl_row_err;
  f.grid = (ctx->abl_rowctas + kErrSlots - 1) / kErrSlots;  // row_err is zero padded
  return f;
}

// One iteration of the two-pass (tiled.hpp:210-229) or four-sweep baseline
// (baseline.hpp:100-110) schedule; see ablation.cuh.
template <typename T>
void launch_ablation_kernels(uot_ctx* ctx) {
  const AblArgs a = abl_args(ctx);
  const dim3 cg(ctx->abl_gx, ctx->abl_gy);
  const unsigned rg = ctx->abl_rowctas, rt = 32 * kAblRowWarps;
  const unsigned fb = finalize_blocks(ctx->pitch);
  if (ctx->variant == UOT_VARIANT_TWO_PASS) {
    abl_row_kernel<true, true, false, T><<<rg, rt, 0, ctx->stream>>>(a);          // part4 -> alpha
    abl_col_kernel<true, false, true, T><<<cg, kAblColThreads, 0, ctx->stream>>>(a);  // part2 -> column partials
    finalize_kernel<kFinIter, true, true><<<fb, kFinThreads, 0, ctx->stream>>>(abl_fin_args(ctx));
    ctx->launches += 3;
  } else {
    abl_col_kernel<false, false, true, T><<<cg, kAblColThreads, 0, ctx->stream>>>(a);  // column sums
    finalize_kernel<kFinSeed, true, true><<<fb, kFinThreads, 0, ctx->stream>>>(abl_fin_args(ctx));  // beta(t)
    abl_col_kernel<false, true, false, T><<<cg, kAblColThreads, 0, ctx->stream>>>(a);  // column scaling
    abl_row_kernel<false, true, false, T><<<rg, rt, 0, ctx->stream>>>(a);             // row sums -> alpha
    abl_row_kernel<false, false, true, T><<<rg, rt, 0, ctx->stream>>>(a);             // row scaling
    abl_baseline_tail_kernel<<<1, 256, 0, ctx->stream>>>(a, rg);
    ctx->launches += 6;
  }
}

int launch_ablation_iteration(uot_ctx* ctx) {
  if (ctx->dtype == UOT_F64)
    launch_ablation_kernels<double>(ctx);
  else
    launch_ablation_kernels<float>(ctx);
  return ctx->cuda(cudaGetLastError(), "ablation launch");
}

// The whole iterate(k) call as one cooperative launch (resident.cuh).
int launch_resident(uot_ctx* ctx, uint64_t k) {
  ResidentArgs r;
  r.P = ctx->Pf();
  r.beta2 = ctx->beta2;
  r.rpd = ctx->rpd;
  r.cpd = ctx->cpd;
  r.alpha = ctx->alpha;
  r.partials = ctx->partials;
  r.col_sums = ctx->col_sums;
  r.bar_flags = ctx->bar_flags;
  r.ctl = ctx->ctl;
  r.rows = ctx->rows;
  r.cols = static_cast<unsigned>(ctx->cols);
  r.pitch = ctx->pitch;
  r.grid = ctx->rgrid;
  r.k = static_cast<unsigned>(std::min<uint64_t>(k, 0xffffffffu));
  r.fi = ctx->fi;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(ctx->rgrid);
  lc.blockDim = dim3(ctx->rcfg->nt);
  lc.dynamicSmemBytes = ctx->rsmem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // grid barriers need every CTA resident
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  ctx->launches++;
  return ctx->cuda(cudaLaunchKernelEx(&lc, ctx->rcfg->fn[ctx->rfull], r), "resident launch");
}

template <int MODE>
int launch_finalize_single(uot_ctx* ctx) {
  const unsigned blocks = finalize_blocks(ctx->pitch);
  ctx->launches++;
  // all of a thread's partial-row loads in flight at once (one L2 round trip),
  // with the smallest register footprint that covers the groups
  const FinalizeArgs f = fin_args(ctx);
  if (ctx->groups <= 5 * kFinSlices)
    finalize_kernel<MODE, true, true, kXchNone, 5><<<blocks, kFinThreads, 0, ctx->stream>>>(f);
  else if (ctx->groups <= 20 * kFinSlices)
    finalize_kernel<MODE, true, true, kXchNone, 20><<<blocks, kFinThreads, 0, ctx->stream>>>(f);
  else
    finalize_kernel<MODE, true, true><<<blocks, kFinThreads, 0, ctx->stream>>>(f);
  return ctx->cuda(cudaGetLastError(), "finalize launch");
}

int nccl_check(uot_ctx* ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return UOT_OK;
  return ctx->fail(UOT_NCCL_ERROR, "%s: %s", what, nccl().GetErrorString(r));
}

// Multi-GPU tail: local reduce -> one exchange of the column sums -> beta.
template <int MODE>
int launch_finalize_dist(uot_ctx* ctx) {
  const unsigned blocks = finalize_blocks(ctx->pitch);
  const FinalizeArgs f = fin_args(ctx);
  ctx->launches += 2;
  if (ctx->xmode == kXchPeer) {  // the allreduce fused into both stages (finalize.cuh)
    if (!ctx->connected) return ctx->fail(UOT_INVALID_PARAMETER, "peer session not connected (uot_peer_connect)");
    finalize_kernel<MODE, true, false, kXchPeer><<<blocks, kFinThreads, 0, ctx->stream>>>(f);
    int rc = ctx->cuda(cudaGetLastError(), "finalize(push) launch");
    if (rc) return rc;
    finalize_kernel<MODE, false, true, kXchPeer><<<blocks, kFinThreads, 0, ctx->stream>>>(f);
    return ctx->cuda(cudaGetLastError(), "finalize(gather) launch");
  }
  finalize_kernel<MODE, true, false, kXchNccl><<<blocks, kFinThreads, 0, ctx->stream>>>(f);
  int rc = ctx->cuda(cudaGetLastError(), "finalize(reduce) launch");
  if (rc) return rc;
  rc = nccl_check(ctx, nccl().AllReduce(ctx->xsum, ctx->xsum, ctx->cols + ctx->nranks, ncclFloat64,
                                        ncclSum, ctx->comm, ctx->stream),
                  "ncclAllReduce");
  if (rc) return rc;
  finalize_kernel<MODE, false, true, kXchNccl><<<blocks, kFinThreads, 0, ctx->stream>>>(f);
  return ctx->cuda(cudaGetLastError(), "finalize(beta) launch");
}

template <int MODE>
int launch_finalize(uot_ctx* ctx) {
  return ctx->xmode != kXchNone ? launch_finalize_dist<MODE>(ctx) : launch_finalize_single<MODE>(ctx);
}

int sync_ctl(uot_ctx* ctx) {
  CK(cudaMemcpyAsync(ctx->h_ctl, ctx->ctl, sizeof(Control), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return UOT_OK;
}

int status_of(uot_ctx* ctx) {
  const int st = ctx->h_ctl->status;
  if (st & kStatusExchangeTimeout)
    return ctx->fail(UOT_CUDA_ERROR, "row-sum exchange timed out (CTAs not co-resident)");
  if (st & kStatusPeerTimeout)
    return ctx->fail(UOT_CUDA_ERROR, "peer exchange timed out (a rank stopped publishing its column sums)");
  if (st & (kStatusDegenerateAlpha | kStatusDegenerateBeta))
    return ctx->fail(UOT_DEGENERATE_SUM, "rescale_factor: %s",
                     (st & kStatusDegenerateAlpha) ? "a row sum is not strictly positive or its factor left the positive finite range"
                                                   : "a column sum is not strictly positive or its factor left the positive finite range");
  return UOT_OK;
}

int check_marginals(uot_ctx* ctx, const double* rpd, const double* cpd, double er, double ep) {
  for (uint64_t i = 0; i < ctx->rows; ++i)
    if (!(rpd[i] > 0.0) || !std::isfinite(rpd[i]))
      return ctx->fail(UOT_INVALID_PARAMETER, "row marginal %llu is not strictly positive",
                       (unsigned long long)(i + ctx->row_offset));
  for (uint64_t j = 0; j < ctx->cols; ++j)
    if (!(cpd[j] > 0.0) || !std::isfinite(cpd[j]))
      return ctx->fail(UOT_INVALID_PARAMETER, "column marginal %llu is not strictly positive",
                       (unsigned long long)j);
  if (uot_compute_fi(er, ep, &ctx->fi) != UOT_OK)
    return ctx->fail(UOT_INVALID_PARAMETER, "er must be positive and finite, ep non-negative and finite");
  return UOT_OK;
}

// Zero the padding columns [cols, pitch) of an uploaded plan.
int pad_after_upload(uot_ctx* ctx) {
  const unsigned gblocks = static_cast<unsigned>(ctx->sms) * 8;
  if (ctx->pitch > ctx->cols) {
    if (ctx->dtype == UOT_F64)
      zero_padding_kernel<<<gblocks, 256, 0, ctx->stream>>>(static_cast<double*>(ctx->P), ctx->rows,
                                                             static_cast<unsigned>(ctx->cols), ctx->pitch);
    else
      zero_padding_kernel<<<gblocks, 256, 0, ctx->stream>>>(ctx->Pf(), ctx->rows, static_cast<unsigned>(ctx->cols),
                                                             ctx->pitch);
    ctx->launches++;
  }
  CK(cudaGetLastError());
  return UOT_OK;
}

int after_matrix_upload(uot_ctx* ctx) {
  int rc = pad_after_upload(ctx);
  if (rc) return rc;
  const unsigned gblocks = static_cast<unsigned>(ctx->sms) * 8;
  CK(cudaMemsetAsync(ctx->dflag, 0, sizeof(int), ctx->stream));
  if (ctx->dtype == UOT_F64)
    validate_matrix_kernel<<<gblocks, 256, 0, ctx->stream>>>(static_cast<const double*>(ctx->P), ctx->rows,
                                                              static_cast<unsigned>(ctx->cols), ctx->pitch, ctx->dflag);
  else
    validate_matrix_kernel<<<gblocks, 256, 0, ctx->stream>>>(ctx->Pf(), ctx->rows, static_cast<unsigned>(ctx->cols),
                                                              ctx->pitch, ctx->dflag);
  ctx->launches++;
  CK(cudaGetLastError());
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, ctx->dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad) return ctx->fail(UOT_INVALID_PARAMETER, "matrix entry is not strictly positive");
  return UOT_OK;
}

int reset_state(uot_ctx* ctx) {
  reset_control_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctl);
  ctx->launches++;
  CK(cudaGetLastError());
  ctx->seeded = false;
  return UOT_OK;
}

void record(uot_ctx* ctx, size_t idx) {
  while (ctx->ev.size() <= idx) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev.push_back(e);
  }
  cudaEventRecord(ctx->ev[idx], ctx->stream);
}

}  // namespace

// ============================================================== C ABI ====
extern "C" {

int uot_create(uot_ctx** out, uint64_t rows, uint64_t cols, int dtype, int device) {
  if (!out) return UOT_INVALID_PARAMETER;
  *out = nullptr;
  auto* ctx = new uot_ctx();
  *out = ctx;
  if (rows < 1 || cols < 1) return ctx->fail(UOT_INVALID_PARAMETER, "matrix must be at least 1x1");
  if (dtype != UOT_F32 && dtype != UOT_F64)
    return ctx->fail(UOT_INVALID_PARAMETER, "dtype %d: neither f32 nor f64 (Dtype, matrix.hpp:13)", dtype);
  ctx->dtype = dtype;
  ctx->esz = dtype == UOT_F64 ? 8 : 4;
  ctx->rows = ctx->global_rows = rows;
  ctx->cols = cols;
  return create_common(ctx, device);
}

int uot_nccl_unique_id(uint8_t* out128) {
  if (!nccl().ok) return UOT_NCCL_ERROR;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return UOT_NCCL_ERROR;
  static_assert(sizeof(id.internal) == 128, "nccl id size");
  std::memcpy(out128, id.internal, 128);
  return UOT_OK;
}

}  // extern "C"

namespace {
// Rank state shared by both exchange flavours (distributed.hpp:65-79).
int create_rank(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, int device, int rank,
                int nranks, const uint64_t* bounds = nullptr) {
  if (!out) return UOT_INVALID_PARAMETER;
  *out = nullptr;
  auto* ctx = new uot_ctx();
  *out = ctx;
  if (global_rows < 1 || cols < 1) return ctx->fail(UOT_INVALID_PARAMETER, "matrix must be at least 1x1");
  if (dtype != UOT_F32 && dtype != UOT_F64)
    return ctx->fail(UOT_INVALID_PARAMETER, "dtype %d: neither f32 nor f64 (Dtype, matrix.hpp:13)", dtype);
  ctx->dtype = dtype;
  ctx->esz = dtype == UOT_F64 ? 8 : 4;
  if (nranks < 1 || static_cast<uint64_t>(nranks) > global_rows)  // plan.cpp:36-39
    return ctx->fail(UOT_PARTITION_ERROR, "RankPartition: %d ranks for %llu rows would leave a rank without rows",
                     nranks, (unsigned long long)global_rows);
  if (rank < 0 || rank >= nranks) return ctx->fail(UOT_PARTITION_ERROR, "rank %d outside [0,%d)", rank, nranks);
  std::vector<uint64_t> b(nranks + 1);
  if (bounds) {  // a caller's RankPartition (distributed.hpp:52-64): contiguous, covering, no empty block
    for (int q = 0; q <= nranks; ++q) b[q] = bounds[q];
    if (b[0] != 0 || b[nranks] != global_rows)
      return ctx->fail(UOT_PARTITION_ERROR, "distributed_solve: partition does not cover the matrix rows");
    for (int q = 0; q < nranks; ++q)
      if (b[q + 1] <= b[q]) return ctx->fail(UOT_PARTITION_ERROR, "partition block %d is empty or unordered", q);
  } else {
    balanced_bounds(nranks, global_rows, b.data());
  }
  ctx->global_rows = global_rows;
  ctx->row_offset = b[rank];
  ctx->rows = b[rank + 1] - b[rank];
  ctx->cols = cols;
  ctx->rank = rank;
  ctx->nranks = nranks;
  ctx->is_dist = true;
  return create_common(ctx, device);
}
}  // namespace

extern "C" {

int uot_create_dist(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, int device,
                    int rank, int nranks, const uint8_t* nccl_id) {
  int rc = create_rank(out, global_rows, cols, dtype, device, rank, nranks);
  if (rc) return rc;
  uot_ctx* ctx = *out;
  // nranks == 1 with an id: a one-rank communicator, so the NCCL exchange path
  // (reduce -> ncclAllReduce -> beta) runs and can be tested on one GPU.
  if (nranks > 1 || nccl_id) {
    ctx->xmode = kXchNccl;
    if (!nccl_id) return ctx->fail(UOT_INVALID_PARAMETER, "a multi-rank session needs the NCCL id of rank 0");
    if (!nccl().ok) return ctx->fail(UOT_NCCL_ERROR, "%s", nccl().err.c_str());
    ncclUniqueId id;
    std::memcpy(id.internal, nccl_id, 128);
    rc = nccl_check(ctx, nccl().CommInitRank(&ctx->comm, nranks, id, rank), "ncclCommInitRank");
    if (rc) return rc;
  }
  return UOT_OK;
}

int create_peer_rank(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, int device, int rank,
                     int nranks, const uint64_t* bounds);

int uot_create_peer(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, int device, int rank,
                    int nranks) {
  return create_peer_rank(out, global_rows, cols, dtype, device, rank, nranks, nullptr);
}

int create_peer_rank(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, int device, int rank,
                     int nranks, const uint64_t* bounds) {
  int rc = create_rank(out, global_rows, cols, dtype, device, rank, nranks, bounds);
  if (rc) return rc;
  uot_ctx* ctx = *out;
  if (nranks > 1) {
    ctx->xmode = kXchPeer;
    ctx->xlen = round_up(static_cast<unsigned>(ctx->cols) + 1, 32);
    ctx->region_bytes = PeerRegion::bytes(nranks, ctx->xlen);
    // cudaMalloc'd so the allocation can be exported with cudaIpcGetMemHandle
    CK(cudaMalloc(reinterpret_cast<void**>(&ctx->region), ctx->region_bytes));
    CK(cudaMemset(ctx->region, 0, ctx->region_bytes));  // flags start at 0; sequence numbers at 1
    CK(cudaMalloc(reinterpret_cast<void**>(&ctx->d_peers), sizeof(unsigned char*) * nranks));
  }
  return UOT_OK;
}

int uot_peer_handle(const uot_ctx* cctx, uint8_t* out64) {
  auto* ctx = const_cast<uot_ctx*>(cctx);
  if (!ctx || !out64) return UOT_INVALID_PARAMETER;
  if (ctx->xmode != kXchPeer) return ctx->fail(UOT_INVALID_PARAMETER, "not a multi-rank peer session");
  CK(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  CK(cudaIpcGetMemHandle(&h, ctx->region));
  std::memcpy(out64, &h, 64);
  return UOT_OK;
}

int uot_peer_connect(uot_ctx* ctx, const uint8_t* handles) {
  if (!ctx || !handles) return UOT_INVALID_PARAMETER;
  if (ctx->xmode != kXchPeer) return ctx->fail(UOT_INVALID_PARAMETER, "not a multi-rank peer session");
  if (ctx->connected) return ctx->fail(UOT_INVALID_PARAMETER, "peer session already connected");
  CK(cudaSetDevice(ctx->device));
  ctx->peer_ptrs.assign(ctx->nranks, nullptr);
  for (int q = 0; q < ctx->nranks; ++q) {
    if (q == ctx->rank) {
      ctx->peer_ptrs[q] = ctx->region;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * static_cast<size_t>(q), 64);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return ctx->fail(UOT_CUDA_ERROR, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
    ctx->peer_ptrs[q] = static_cast<unsigned char*>(p);
  }
  CK(cudaMemcpy(ctx->d_peers, ctx->peer_ptrs.data(), sizeof(unsigned char*) * ctx->nranks,
                cudaMemcpyHostToDevice));
  ctx->connected = true;
  return UOT_OK;
}

int uot_exchange_mode(const uot_ctx* ctx) { return ctx ? ctx->xmode : -1; }

int uot_set_schedule(uot_ctx* ctx, int schedule) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  if (schedule != UOT_SCHEDULE_UNIFORM && schedule != UOT_SCHEDULE_WEIGHTED && schedule != UOT_SCHEDULE_DYNAMIC)
    return ctx->fail(UOT_INVALID_PARAMETER, "unknown row-batch schedule %d", schedule);
  if (schedule == UOT_SCHEDULE_WEIGHTED && (!ctx->pinned || ctx->weights.size() != ctx->groups))
    return ctx->fail(UOT_CONFIG_ERROR, "the weighted schedule needs one sweep CTA per SM and group weights "
                                       "(uot_set_group_weights / uot_calibrate_schedule)");
  ctx->schedule = schedule;
  ctx->dyn = schedule == UOT_SCHEDULE_DYNAMIC && !ctx->wide ? 1 : 0;
  return UOT_OK;
}

int uot_set_deterministic(uot_ctx* ctx, int on) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  if (on) return uot_set_schedule(ctx, ctx->weights.size() == ctx->groups && ctx->pinned ? UOT_SCHEDULE_WEIGHTED
                                                                                        : UOT_SCHEDULE_UNIFORM);
  return uot_set_schedule(ctx, UOT_SCHEDULE_DYNAMIC);
}

int uot_set_group_weights(uot_ctx* ctx, const uint32_t* w, uint32_t n) {
  if (!ctx || !w) return UOT_INVALID_PARAMETER;
  if (!ctx->pinned)
    return ctx->fail(UOT_CONFIG_ERROR, "weighted row blocks need one sweep CTA on every SM (grid %u, %d SMs)",
                     ctx->grid, ctx->sms);
  if (n != ctx->groups) return ctx->fail(UOT_INVALID_PARAMETER, "%u weights for %u row groups", n, ctx->groups);
  uint64_t sum = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (w[i] < 1 || w[i] > (1u << 20)) return ctx->fail(UOT_INVALID_PARAMETER, "group weight %u out of [1, 2^20]", w[i]);
    sum += w[i];
  }
  ctx->weights.assign(w, w + n);
  const auto b = weighted_bounds(ctx->rows, ctx->weights);
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(ctx->d_gbounds, b.data(), sizeof(unsigned long long) * b.size(), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return uot_set_schedule(ctx, UOT_SCHEDULE_WEIGHTED);
}

int uot_get_schedule_stats(const uot_ctx* cctx, uint32_t* cta_smid, uint32_t* cta_batches, uint32_t* group_weight) {
  auto* ctx = const_cast<uot_ctx*>(cctx);
  if (!ctx) return UOT_INVALID_PARAMETER;
  CK(cudaSetDevice(ctx->device));
  std::vector<unsigned> h(kDbg * static_cast<size_t>(ctx->grid));
  CK(cudaMemcpyAsync(h.data(), ctx->d_dbg, sizeof(unsigned) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (unsigned c = 0; c < ctx->grid; ++c) {
    if (cta_smid) cta_smid[c] = h[kDbg * c];
    if (cta_batches) cta_batches[c] = h[kDbg * c + 1];
  }
  if (group_weight)
    for (unsigned g = 0; g < ctx->groups; ++g)
      group_weight[g] = ctx->weights.size() == ctx->groups ? ctx->weights[g] : 1u;
  return UOT_OK;
}

// Calibration of the weighted schedule, on a scratch copy of the plan (the
// session's plan, factors, column sums and stop state are untouched; only
// never-reset exchange tags advance):
//   1. `k` dynamic iterations: the row batches each group took are its first
//      weight (the per-SM HBM rates the dynamic counter adapts to);
//   2. kRefineRounds rounds of two iterations under the weighted schedule
//      itself: each group's completion time (its CTAs' last store, from the
//      earliest CTA start) rescales its weight by (mean time / its time)^0.75,
//      so the static blocks finish together as the dynamic batches do.
// Deterministic afterwards: the weights are fixed, so every later solve with
// them is bit-reproducible.
constexpr int kRefineRounds = 3;  // (measured: 6 or 10 rounds, or an undamped update, are no better)
int uot_calibrate_schedule(uot_ctx* ctx, uint32_t k) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  if (!ctx->have_problem || !ctx->seeded)
    return ctx->fail(UOT_INVALID_PARAMETER, "calibration needs a problem and its column sums (init_col_sums)");
  if (!ctx->pinned)
    return ctx->fail(UOT_CONFIG_ERROR, "weighted row blocks need one sweep CTA on every SM (grid %u, %d SMs)",
                     ctx->grid, ctx->sms);
  if (ctx->variant != UOT_VARIANT_FUSED || ctx->wide)
    return ctx->fail(UOT_CONFIG_ERROR, "calibration runs the fused sweep");
  k = std::max<uint32_t>(2, std::min<uint32_t>(k, 64));
  CK(cudaSetDevice(ctx->device));
  const size_t pbytes = static_cast<size_t>(ctx->rows) * ctx->pitch * ctx->esz;
  void* scratch = nullptr;
  if (cudaMalloc(&scratch, pbytes) != cudaSuccess) {
    cudaGetLastError();
    return ctx->fail(UOT_CONFIG_ERROR, "not enough device memory for a calibration copy of the plan (%zu bytes)",
                     pbytes);
  }
  // saved state: factors, column sums, control
  std::vector<double> sb(2 * static_cast<size_t>(ctx->pitch)), sc(ctx->cols), sa(ctx->rows);
  Control* saved = nullptr;
  int rc = ctx->cuda(cudaMalloc(reinterpret_cast<void**>(&saved), sizeof(Control)), "cudaMalloc");
  if (!rc) rc = ctx->cuda(cudaMemcpyAsync(scratch, ctx->P, pbytes, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
  if (!rc) rc = ctx->cuda(cudaMemcpyAsync(saved, ctx->ctl, sizeof(Control), cudaMemcpyDeviceToDevice, ctx->stream), "copy");
  if (!rc) rc = ctx->cuda(cudaMemcpyAsync(sb.data(), ctx->beta2, sb.size() * 8, cudaMemcpyDeviceToHost, ctx->stream), "copy");
  if (!rc) rc = ctx->cuda(cudaMemcpyAsync(sc.data(), ctx->col_sums, sc.size() * 8, cudaMemcpyDeviceToHost, ctx->stream), "copy");
  if (!rc) rc = ctx->cuda(cudaMemcpyAsync(sa.data(), ctx->alpha, sa.size() * 8, cudaMemcpyDeviceToHost, ctx->stream), "copy");
  void* real = ctx->P;
  const int sched = ctx->schedule, dyn = ctx->dyn;
  std::vector<uint64_t> counts(ctx->groups, 0);
  std::vector<double> wd(ctx->groups, 1.0);
  auto to_weights = [&]() {  // integer weights in [1, 2^19] proportional to wd
    double m = 0.0;
    for (double x : wd) m = std::max(m, x);
    std::vector<uint32_t> w(ctx->groups);
    for (unsigned g = 0; g < ctx->groups; ++g)
      w[g] = static_cast<uint32_t>(std::max(1.0, std::min(double(1u << 19), std::round(wd[g] / m * (1u << 19)))));
    return w;
  };
  if (!rc) {
    ctx->P = scratch;
    ctx->schedule = UOT_SCHEDULE_DYNAMIC;
    ctx->dyn = 1;
    begin_iterate_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctl, 1e-300);
    std::vector<unsigned> h(kDbg * static_cast<size_t>(ctx->grid));
    auto one_iteration = [&]() {
      rc = launch_sweep(ctx, false);
      if (!rc) rc = launch_finalize_single<kFinIter>(ctx);  // local finalize: no peer exchange for a scratch run
      if (!rc) rc = ctx->cuda(cudaMemcpyAsync(h.data(), ctx->d_dbg, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream), "copy");
      if (!rc) rc = ctx->cuda(cudaStreamSynchronize(ctx->stream), "calibration sweep");
    };
    for (uint32_t i = 0; i < k && !rc; ++i) {
      one_iteration();
      if (i == 0) continue;  // warm-up
      for (unsigned g = 0; g < ctx->groups && !rc; ++g) counts[g] += h[kDbg * (g * ctx->G) + 1];
    }
    for (unsigned g = 0; g < ctx->groups; ++g) wd[g] = static_cast<double>(std::max<uint64_t>(1, counts[g]));
    ctx->schedule = UOT_SCHEDULE_WEIGHTED;
    ctx->dyn = 0;
    for (int round = 0; round < kRefineRounds && !rc; ++round) {
      const auto b = weighted_bounds(ctx->rows, to_weights());
      rc = ctx->cuda(cudaMemcpyAsync(ctx->d_gbounds, b.data(), sizeof(unsigned long long) * b.size(),
                                     cudaMemcpyHostToDevice, ctx->stream), "copy");
      for (int i = 0; i < 2 && !rc; ++i) one_iteration();  // the second one is measured
      if (rc) break;
      unsigned t0 = h[2];
      for (unsigned c = 1; c < ctx->grid; ++c)
        if (static_cast<int>(h[kDbg * c + 2] - t0) < 0) t0 = h[kDbg * c + 2];
      std::vector<double> tg(ctx->groups, 0.0);
      double tmean = 0.0;
      for (unsigned g = 0; g < ctx->groups; ++g) {
        for (unsigned c = g * ctx->G; c < (g + 1) * ctx->G; ++c)
          tg[g] = std::max(tg[g], static_cast<double>(static_cast<int>(h[kDbg * c + 3] - t0)));
        tg[g] = std::max(tg[g], 1.0);
        tmean += tg[g] / ctx->groups;
      }
      for (unsigned g = 0; g < ctx->groups; ++g) wd[g] *= std::pow(tmean / tg[g], 0.75);
    }
    ctx->P = real;
    ctx->schedule = sched;
    ctx->dyn = dyn;
  }
  if (!rc) rc = ctx->cuda(cudaMemcpyAsync(ctx->beta2, sb.data(), sb.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "copy");
  if (!rc) rc = ctx->cuda(cudaMemcpyAsync(ctx->col_sums, sc.data(), sc.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "copy");
  if (!rc) rc = ctx->cuda(cudaMemcpyAsync(ctx->alpha, sa.data(), sa.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "copy");
  if (!rc) {
    restore_control_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctl, saved);
    ctx->launches++;
    rc = ctx->cuda(cudaStreamSynchronize(ctx->stream), "calibration restore");
  }
  cudaFree(scratch);
  if (saved) cudaFree(saved);
  if (rc) return rc;
  if ((rc = sync_ctl(ctx))) return rc;
  const auto w = to_weights();
  return uot_set_group_weights(ctx, w.data(), ctx->groups);
}

int uot_get_group_weights(const uot_ctx* ctx, uint32_t* w, uint32_t n) {
  if (!ctx || !w) return UOT_INVALID_PARAMETER;
  if (ctx->weights.size() != ctx->groups || n < ctx->groups) return UOT_INVALID_PARAMETER;
  std::copy(ctx->weights.begin(), ctx->weights.end(), w);
  return UOT_OK;
}

int uot_set_resident(uot_ctx* ctx, int on) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  ctx->resident_on = on != 0;
  return UOT_OK;
}

int uot_set_variant(uot_ctx* ctx, int variant) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  if (variant != UOT_VARIANT_FUSED && variant != UOT_VARIANT_TWO_PASS && variant != UOT_VARIANT_BASELINE)
    return ctx->fail(UOT_INVALID_PARAMETER, "unknown iteration variant %d", variant);
  if (variant != UOT_VARIANT_FUSED && ctx->nranks > 1)
    return ctx->fail(UOT_INVALID_PARAMETER, "the ablation schedules are single-GPU only");
  if (variant != UOT_VARIANT_TWO_PASS && ctx->wide)
    return ctx->fail(UOT_CONFIG_ERROR, "rows of %llu columns exceed one slice per SM: two-pass schedule only",
                     (unsigned long long)ctx->cols);
  CK(cudaSetDevice(ctx->device));
  if (variant != UOT_VARIANT_FUSED && !ctx->abl_partials) {
    ctx->abl_gx = ((ctx->pitch + 3) / 4 + kAblColThreads * kAblColV - 1) / (kAblColThreads * kAblColV);
    ctx->abl_gy = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>(ctx->rows, (4u * ctx->sms + ctx->abl_gx - 1) / ctx->abl_gx)));
    ctx->abl_rowctas = static_cast<unsigned>((ctx->rows + kAblRowWarps - 1) / kAblRowWarps);
    const size_t nerr = (ctx->abl_rowctas + kErrSlots - 1) / kErrSlots * kErrSlots;
    int rc;
    if ((rc = dalloc(ctx, &ctx->abl_partials, static_cast<size_t>(ctx->abl_gy) * ctx->pitch))) return rc;
    if ((rc = dalloc(ctx, &ctx->abl_row_err, nerr))) return rc;
    CK(cudaMemsetAsync(ctx->abl_row_err, 0, nerr * sizeof(double), ctx->stream));
  }
  ctx->variant = variant;
  return UOT_OK;
}

void uot_destroy(uot_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
  }
  if (ctx->comm) nccl().CommDestroy(ctx->comm);
  if (!ctx->group_local)
    for (int q = 0; q < static_cast<int>(ctx->peer_ptrs.size()); ++q)
      if (q != ctx->rank && ctx->peer_ptrs[q]) cudaIpcCloseMemHandle(ctx->peer_ptrs[q]);
  if (ctx->xev) cudaEventDestroy(ctx->xev);
  if (ctx->region) cudaFree(ctx->region);
  if (ctx->d_peers) cudaFree(ctx->d_peers);
  for (auto e : ctx->ev) cudaEventDestroy(e);
  void* bufs[] = {ctx->P,     ctx->rpd,   ctx->cpd,      ctx->alpha,   ctx->beta2, ctx->col_sums, ctx->xsum,
                  ctx->partials, ctx->cta_err, ctx->xrec, ctx->mail, ctx->d_dbg, ctx->d_slot, ctx->d_gbounds, ctx->ctl, ctx->dflag, ctx->bar_flags,
                  ctx->abl_partials, ctx->abl_row_err};
  for (void* p : bufs)
    if (p) cudaFree(p);
  if (ctx->h_ctl) cudaFreeHost(ctx->h_ctl);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* uot_last_error(const uot_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null session"; }

int uot_get_layout(const uot_ctx* ctx, uot_layout* o) {
  if (!ctx || !o || !ctx->cfg) return UOT_INVALID_PARAMETER;
  o->rows = ctx->rows;
  o->cols = ctx->cols;
  o->row_offset = ctx->row_offset;
  o->global_rows = ctx->global_rows;
  o->pitch = ctx->pitch;
  o->slice = ctx->slice;
  o->G = ctx->G;
  o->groups = ctx->groups;
  o->rows_per_step = ctx->B;
  o->threads = ctx->cfg->nt + 32 * (1 + ctx->cfg->nf);
  o->chunks = ctx->cfg->v;
  o->smem_bytes = static_cast<uint32_t>(ctx->smem);
  o->resident = ctx->rcfg && ctx->resident_on && ctx->xmode == kXchNone ? 1 : 0;
  o->dtype = ctx->dtype;
  o->dynamic = ctx->dyn;
  o->schedule = ctx->schedule;
  o->pinned = ctx->pinned ? 1 : 0;
  o->nbuf = ctx->cfg->nbuf;
  o->sms = ctx->sms;
  o->rank = ctx->rank;
  o->nranks = ctx->nranks;
  o->device = ctx->device;
  o->evict_first = ctx->evict_first;
  o->smid_map = ctx->smid_map;
  o->exchange = ctx->xmode;
  o->variant = ctx->variant;
  o->keep_batches = ctx->dyn ? 0u : ctx->keep;
  return UOT_OK;
}

void* uot_get_stream(const uot_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

}  // extern "C"

namespace {
int dtype_check(uot_ctx* ctx, int want, const char* who) {
  if (ctx->dtype == want) return UOT_OK;
  return ctx->fail(UOT_INVALID_PARAMETER, "%s: the session holds a Problem<%s>", who,
                   ctx->dtype == UOT_F64 ? "double" : "float");
}

int set_problem_any(uot_ctx* ctx, const void* a, const double* rpd, const double* cpd, double er, double ep) {
  CK(cudaSetDevice(ctx->device));
  int rc = check_marginals(ctx, rpd, cpd, er, ep);
  if (rc) return rc;
  ctx->er = er;
  ctx->ep = ep;
  ctx->have_problem = false;
  CK(cudaMemcpy2DAsync(ctx->P, ctx->pitch * ctx->esz, a, ctx->cols * ctx->esz, ctx->cols * ctx->esz, ctx->rows,
                       cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->rpd, rpd, ctx->rows * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->cpd, cpd, ctx->cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  if ((rc = reset_state(ctx))) return rc;
  if ((rc = after_matrix_upload(ctx))) return rc;
  ctx->have_problem = true;
  return UOT_OK;
}

int set_plan_any(uot_ctx* ctx, const void* a) {
  if (!ctx->have_problem) return ctx->fail(UOT_INVALID_PARAMETER, "no problem set");
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpy2DAsync(ctx->P, ctx->pitch * ctx->esz, a, ctx->cols * ctx->esz, ctx->cols * ctx->esz, ctx->rows,
                       cudaMemcpyHostToDevice, ctx->stream));
  return after_matrix_upload(ctx);
}

int get_plan_any(uot_ctx* ctx, void* out) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpy2DAsync(out, ctx->cols * ctx->esz, ctx->P, ctx->pitch * ctx->esz, ctx->cols * ctx->esz, ctx->rows,
                       cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return UOT_OK;
}
}  // namespace

extern "C" {

int uot_set_problem(uot_ctx* ctx, const float* a, const double* rpd, const double* cpd, double er,
                    double ep) {
  if (!ctx || !a || !rpd || !cpd) return UOT_INVALID_PARAMETER;
  int rc = dtype_check(ctx, UOT_F32, "uot_set_problem");
  return rc ? rc : set_problem_any(ctx, a, rpd, cpd, er, ep);
}

int uot_set_problem_f64(uot_ctx* ctx, const double* a, const double* rpd, const double* cpd, double er,
                        double ep) {
  if (!ctx || !a || !rpd || !cpd) return UOT_INVALID_PARAMETER;
  int rc = dtype_check(ctx, UOT_F64, "uot_set_problem_f64");
  return rc ? rc : set_problem_any(ctx, a, rpd, cpd, er, ep);
}

int uot_generate_problem(uot_ctx* ctx, uint64_t seed, double er, double ep) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  CK(cudaSetDevice(ctx->device));
  if (uot_compute_fi(er, ep, &ctx->fi) != UOT_OK)
    return ctx->fail(UOT_INVALID_PARAMETER, "er must be positive and finite, ep non-negative and finite");
  ctx->er = er;
  ctx->ep = ep;
  ctx->have_problem = false;
  const unsigned gblocks = static_cast<unsigned>(ctx->sms) * 16;
  if (ctx->dtype == UOT_F64)
    gen_matrix_kernel<<<gblocks, 256, 0, ctx->stream>>>(static_cast<double*>(ctx->P), seed, ctx->row_offset,
                                                       ctx->rows, static_cast<unsigned>(ctx->cols), ctx->pitch);
  else
    gen_matrix_kernel<<<gblocks, 256, 0, ctx->stream>>>(ctx->Pf(), seed, ctx->row_offset, ctx->rows,
                                                       static_cast<unsigned>(ctx->cols), ctx->pitch);
  gen_marginals_kernel<<<gblocks, 256, 0, ctx->stream>>>(ctx->rpd, ctx->cpd, seed, ctx->global_rows,
                                                         ctx->row_offset, ctx->rows,
                                                         static_cast<unsigned>(ctx->cols));
  ctx->launches += 2;
  CK(cudaGetLastError());
  int rc = reset_state(ctx);
  if (rc) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->have_problem = true;
  return UOT_OK;
}

int uot_set_fi(uot_ctx* ctx, double fi) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  if (!(fi > 0.0) || !(fi <= 1.0)) return ctx->fail(UOT_INVALID_PARAMETER, "fi must lie in (0, 1]");
  ctx->fi = fi;
  return UOT_OK;
}

int uot_set_iterate_input(uot_ctx* ctx, const void* a, int dtype, const double* rpd, const double* cpd,
                          double fi) {
  if (!ctx || !a || !rpd || !cpd) return UOT_INVALID_PARAMETER;
  int rc = dtype_check(ctx, dtype, "uot_set_iterate_input");
  if (rc) return rc;
  if (!std::isfinite(fi)) return ctx->fail(UOT_INVALID_PARAMETER, "fi must be finite");
  CK(cudaSetDevice(ctx->device));
  ctx->have_problem = false;
  CK(cudaMemcpy2DAsync(ctx->P, ctx->pitch * ctx->esz, a, ctx->cols * ctx->esz, ctx->cols * ctx->esz, ctx->rows,
                       cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->rpd, rpd, ctx->rows * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->cpd, cpd, ctx->cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  if ((rc = reset_state(ctx))) return rc;
  if ((rc = pad_after_upload(ctx))) return rc;
  ctx->fi = fi;
  ctx->have_problem = true;
  return UOT_OK;
}

int uot_set_plan(uot_ctx* ctx, const float* a) {
  if (!ctx || !a) return UOT_INVALID_PARAMETER;
  int rc = dtype_check(ctx, UOT_F32, "uot_set_plan");
  return rc ? rc : set_plan_any(ctx, a);
}

int uot_set_plan_f64(uot_ctx* ctx, const double* a) {
  if (!ctx || !a) return UOT_INVALID_PARAMETER;
  int rc = dtype_check(ctx, UOT_F64, "uot_set_plan_f64");
  return rc ? rc : set_plan_any(ctx, a);
}

int uot_init_col_sums(uot_ctx* ctx) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  if (ctx->group_local && ctx->nranks > 1)
    return ctx->fail(UOT_INVALID_PARAMETER, "a rank of a session group: use uot_group_init_col_sums");
  if (!ctx->have_problem) return ctx->fail(UOT_INVALID_PARAMETER, "no problem set");
  CK(cudaSetDevice(ctx->device));
  int rc = reset_state(ctx);
  if (rc) return rc;
  if (ctx->wide) {  // column sums with the two-pass schedule's column kernel (baseline.hpp:30-38)
    const dim3 cg(ctx->abl_gx, ctx->abl_gy);
    if (ctx->dtype == UOT_F64)
      abl_col_kernel<false, false, true, double><<<cg, kAblColThreads, 0, ctx->stream>>>(abl_args(ctx));
    else
      abl_col_kernel<false, false, true, float><<<cg, kAblColThreads, 0, ctx->stream>>>(abl_args(ctx));
    finalize_kernel<kFinSeed, true, true><<<finalize_blocks(ctx->pitch), kFinThreads, 0, ctx->stream>>>(
        abl_fin_args(ctx));
    ctx->launches += 2;
    CK(cudaGetLastError());
  } else {
    if ((rc = launch_sweep(ctx, /*seed=*/true))) return rc;
    if ((rc = launch_finalize<kFinSeed>(ctx))) return rc;
  }
  if ((rc = sync_ctl(ctx))) return rc;
  ctx->seeded = true;
  return UOT_OK;
}

int uot_set_col_sums(uot_ctx* ctx, const double* col_sums) {
  if (!ctx || !col_sums) return UOT_INVALID_PARAMETER;
  if (!ctx->have_problem) return ctx->fail(UOT_INVALID_PARAMETER, "no problem set");
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(ctx->col_sums, col_sums, ctx->cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  // A new FusedState re-opens a session that stopped on convergence (a failed
  // one stays stopped): without this the beta-only finalize below would skip.
  resume_control_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctl);
  ctx->launches++;
  // Recompute beta(iter+1) from the given state; its error slot starts at zero.
  CK(cudaMemsetAsync(reinterpret_cast<char*>(ctx->ctl) + offsetof(Control, err_beta), 0,
                     2 * sizeof(double), ctx->stream));
  const unsigned blocks = finalize_blocks(ctx->pitch);
  ctx->launches++;
  finalize_kernel<kFinBetaOnly, false, true><<<blocks, kFinThreads, 0, ctx->stream>>>(fin_args(ctx));
  CK(cudaGetLastError());
  int rc = sync_ctl(ctx);
  if (rc) return rc;
  ctx->seeded = true;
  return UOT_OK;
}

int uot_get_col_sums(const uot_ctx* cctx, double* out) {
  auto* ctx = const_cast<uot_ctx*>(cctx);
  if (!ctx || !out) return UOT_INVALID_PARAMETER;
  if (!ctx->seeded) return ctx->fail(UOT_INVALID_PARAMETER, "no carried column sums (call init_col_sums)");
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(out, ctx->col_sums, ctx->cols * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return UOT_OK;
}

int uot_iterate(uot_ctx* ctx, uint64_t k, double tol, uint64_t* iterations, double* final_error,
                int* converged) {
  return uot_iterate_timed(ctx, k, tol, iterations, final_error, converged, nullptr);
}

int uot_synchronize(uot_ctx* ctx) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  return UOT_OK;
}

int uot_iterate_timed(uot_ctx* ctx, uint64_t k, double tol, uint64_t* iterations, double* final_error,
                      int* converged, double* device_ms) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  if (ctx->group_local && ctx->nranks > 1)
    return ctx->fail(UOT_INVALID_PARAMETER, "a rank of a session group: use uot_group_iterate");
  if (!ctx->have_problem) return ctx->fail(UOT_INVALID_PARAMETER, "no problem set");
  if (!ctx->seeded)
    return ctx->fail(UOT_INVALID_PARAMETER, "carried column sums missing (call init_col_sums)");
  if (!(tol > 0.0)) return ctx->fail(UOT_INVALID_PARAMETER, "tol must be positive");
  if (k < 1) return ctx->fail(UOT_INVALID_PARAMETER, "max_iter must be at least 1");
  CK(cudaSetDevice(ctx->device));
  const uint64_t before = ctx->h_ctl->iter;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (device_ms) {
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    CK(cudaEventRecord(t0, ctx->stream));
  }
  begin_iterate_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ctl, tol);
  ctx->launches++;
  CK(cudaGetLastError());
  int rc;
  const bool resident =
      ctx->rcfg != nullptr && ctx->resident_on && ctx->xmode == kXchNone && ctx->variant == UOT_VARIANT_FUSED;
  if (ctx->variant != UOT_VARIANT_FUSED) {
    for (uint64_t i = 0; i < k; ++i) {
      if (ctx->timing) record(ctx, 3 * i);
      if ((rc = launch_ablation_iteration(ctx))) return rc;
      if (ctx->timing) record(ctx, 3 * i + 1);
      if (ctx->timing) record(ctx, 3 * i + 2);
    }
  } else if (resident) {  // k iterations, one launch: sweeps, reductions, stop test inside
    if (ctx->timing) record(ctx, 0);
    if ((rc = launch_resident(ctx, k))) return rc;
    if (ctx->timing) record(ctx, 1);
  } else {
    for (uint64_t i = 0; i < k; ++i) {
      if (ctx->timing) record(ctx, 3 * i);
      if ((rc = launch_sweep(ctx, false))) return rc;
      if (ctx->timing) record(ctx, 3 * i + 1);
      if ((rc = launch_finalize<kFinIter>(ctx))) return rc;
      if (ctx->timing) record(ctx, 3 * i + 2);
    }
  }
  if (device_ms) CK(cudaEventRecord(t1, ctx->stream));
  if ((rc = sync_ctl(ctx))) return rc;
  if (device_ms) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, t0, t1));
    *device_ms = ms;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  if (ctx->timing) {
    ctx->sweep_ms = ctx->fin_ms = 0.0;
    if (resident) {  // one launch: reported as sweep time, no separate finalize
      float a = 0.f;
      cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
      ctx->sweep_ms = a;
    }
    for (uint64_t i = 0; i < (resident ? 0 : k); ++i) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, ctx->ev[3 * i], ctx->ev[3 * i + 1]);
      cudaEventElapsedTime(&b, ctx->ev[3 * i + 1], ctx->ev[3 * i + 2]);
      ctx->sweep_ms += a;
      ctx->fin_ms += b;
    }
    ctx->sweeps_timed = resident ? std::max<uint64_t>(1, ctx->h_ctl->iter - before) : k;
  }
  if (iterations) *iterations = ctx->h_ctl->iter - before;
  if (final_error) *final_error = ctx->h_ctl->last_error;
  if (converged) *converged = ctx->h_ctl->converged;
  return status_of(ctx);
}

int uot_get_factors(const uot_ctx* cctx, double* alpha, double* beta) {
  auto* ctx = const_cast<uot_ctx*>(cctx);
  if (!ctx) return UOT_INVALID_PARAMETER;
  const uint64_t it = ctx->h_ctl ? ctx->h_ctl->iter : 0;
  if (it == 0) return ctx->fail(UOT_INVALID_PARAMETER, "no completed iteration");
  CK(cudaSetDevice(ctx->device));
  if (alpha)
    CK(cudaMemcpyAsync(alpha, ctx->alpha, ctx->rows * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  if (beta)
    CK(cudaMemcpyAsync(beta, ctx->beta2 + (it & 1ull) * ctx->pitch, ctx->cols * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return UOT_OK;
}

int uot_get_plan(const uot_ctx* cctx, float* out) {
  auto* ctx = const_cast<uot_ctx*>(cctx);
  if (!ctx || !out) return UOT_INVALID_PARAMETER;
  int rc = dtype_check(ctx, UOT_F32, "uot_get_plan");
  return rc ? rc : get_plan_any(ctx, out);
}

int uot_get_plan_f64(const uot_ctx* cctx, double* out) {
  auto* ctx = const_cast<uot_ctx*>(cctx);
  if (!ctx || !out) return UOT_INVALID_PARAMETER;
  int rc = dtype_check(ctx, UOT_F64, "uot_get_plan_f64");
  return rc ? rc : get_plan_any(ctx, out);
}

int uot_get_report(const uot_ctx* ctx, uint64_t* iterations, double* final_error, int* converged) {
  if (!ctx || !ctx->h_ctl) return UOT_INVALID_PARAMETER;
  if (iterations) *iterations = ctx->h_ctl->iter;
  if (final_error) *final_error = ctx->h_ctl->last_error;
  if (converged) *converged = ctx->h_ctl->converged;
  return UOT_OK;
}

int uot_get_comm_stats(const uot_ctx* ctx, uint64_t* calls, uint64_t* doubles) {
  if (!ctx || !ctx->h_ctl) return UOT_INVALID_PARAMETER;
  // One allreduce of the column vector per completed iteration (distributed.hpp:88-94).
  const uint64_t it = ctx->is_dist ? ctx->h_ctl->iter : 0;
  if (calls) *calls = it;
  if (doubles) *doubles = it * ctx->cols;
  return UOT_OK;
}

int uot_set_timing(uot_ctx* ctx, int enabled) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  ctx->timing = enabled != 0;
  return UOT_OK;
}

int uot_get_timing(const uot_ctx* ctx, double* sweep_ms, double* finalize_ms, uint64_t* sweeps) {
  if (!ctx) return UOT_INVALID_PARAMETER;
  if (sweep_ms) *sweep_ms = ctx->sweep_ms;
  if (finalize_ms) *finalize_ms = ctx->fin_ms;
  if (sweeps) *sweeps = ctx->sweeps_timed;
  return UOT_OK;
}

uint64_t uot_kernel_launches(const uot_ctx* ctx) { return ctx ? ctx->launches : 0; }

// Phase timers of the trace build (-DUOT_TRACE); returns UOT_CONFIG_ERROR otherwise.
UOT_API int uot_trace_read(unsigned long long* out32, int reset) {
#ifdef UOT_TRACE
  if (cudaMemcpyFromSymbol(out32, uot_trace, 32 * sizeof(unsigned long long)) != cudaSuccess) return UOT_CUDA_ERROR;
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(uot_trace, z, sizeof(z));
  }
  return UOT_OK;
#else
  (void)out32;
  (void)reset;
  return UOT_CONFIG_ERROR;
#endif
}

// Pinned host staging for callers that feed the session from host memory.
void* uot_host_alloc(uint64_t bytes) {
  void* p = nullptr;
  return cudaMallocHost(&p, std::max<uint64_t>(bytes, 1)) == cudaSuccess ? p : nullptr;
}
void uot_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

// ------------------------------------------------------------ host scalars --
int uot_compute_fi(double er, double ep, double* fi) {  // scaling.cpp:9-13
  if (!(er > 0.0) || !std::isfinite(er)) return UOT_INVALID_PARAMETER;
  if (!(ep >= 0.0) || !std::isfinite(ep)) return UOT_INVALID_PARAMETER;
  *fi = er / (er + ep);
  return UOT_OK;
}

int uot_rescale_factor(double target, double sum, double fi, double* out) {  // scaling.cpp:15-22
  if (!(sum > 0.0)) return UOT_DEGENERATE_SUM;
  const double f = std::pow(target / sum, fi);
  if (!(f > 0.0) || !std::isfinite(f)) return UOT_DEGENERATE_SUM;
  *out = f;
  return UOT_OK;
}

double uot_convergence_error(const double* alpha, uint64_t m, const double* beta, uint64_t n) {
  double e = 0.0;  // scaling.cpp:24-29
  for (uint64_t i = 0; i < m; ++i) e = std::max(e, std::abs(alpha[i] - 1.0));
  for (uint64_t j = 0; j < n; ++j) e = std::max(e, std::abs(beta[j] - 1.0));
  return e;
}

int uot_rank_partition(uint64_t ranks, uint64_t rows, uint64_t* bounds) {  // plan.cpp:35-44
  if (ranks < 1 || ranks > rows) return UOT_PARTITION_ERROR;
  balanced_bounds(ranks, rows, bounds);
  return UOT_OK;
}

int uot_gen_block_f32(uint64_t seed, uint64_t global_rows, uint64_t n, uint64_t row0, uint64_t rows,
                      float* a, double* rpd, double* cpd, int threads) {  // problem_io.hpp:17-31
  if (global_rows < 1 || n < 1 || row0 + rows > global_rows) return UOT_INVALID_PARAMETER;
  auto unit_at = [seed](uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return static_cast<double>((z >> 11) + 1) * 0x1p-53;
  };
  const uint64_t mn = rows * n, first = row0 * n, gmn = global_rows * n;
  const int nt = std::max(1, std::min<int>(threads, 256));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (uint64_t k = mn * t / nt; k < mn * (t + 1) / nt; ++k) a[k] = static_cast<float>(unit_at(first + k));
    });
  for (auto& x : th) x.join();
  if (rpd)
    for (uint64_t i = 0; i < rows; ++i) rpd[i] = unit_at(gmn + row0 + i);
  if (cpd)
    for (uint64_t j = 0; j < n; ++j) cpd[j] = unit_at(gmn + global_rows + j);
  return UOT_OK;
}

int uot_gen_block_f64(uint64_t seed, uint64_t global_rows, uint64_t n, uint64_t row0, uint64_t rows,
                      double* a, double* rpd, double* cpd, int threads) {  // gen_problem_t<double>
  if (global_rows < 1 || n < 1 || row0 + rows > global_rows) return UOT_INVALID_PARAMETER;
  auto unit_at = [seed](uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return static_cast<double>((z >> 11) + 1) * 0x1p-53;
  };
  const uint64_t mn = rows * n, first = row0 * n, gmn = global_rows * n;
  const int nt = std::max(1, std::min<int>(threads, 256));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (uint64_t k = mn * t / nt; k < mn * (t + 1) / nt; ++k) a[k] = unit_at(first + k);
    });
  for (auto& x : th) x.join();
  if (rpd)
    for (uint64_t i = 0; i < rows; ++i) rpd[i] = unit_at(gmn + row0 + i);
  if (cpd)
    for (uint64_t j = 0; j < n; ++j) cpd[j] = unit_at(gmn + global_rows + j);
  return UOT_OK;
}

int uot_gen_problem_f32(uint64_t seed, uint64_t m, uint64_t n, float* a, double* rpd, double* cpd,
                        int threads) {
  return uot_gen_block_f32(seed, m, n, 0, m, a, rpd, cpd, threads);
}

}  // extern "C"

// ==================================================== .uotp problem files ====
// The reference's container (problem_io.cpp:13-141): 40-byte little-endian
// header {"UOTP", u16 version 1, u16 dtype (1 f32, 2 f64), u64 M, u64 N, f64 er,
// f64 ep}, then A row-major, rpd (M f64), cpd (N f64); the file size must equal
// the header's extents exactly. Sessions stream THEIR row block between the file
// and HBM through two page-locked staging buffers (read/write overlapped with
// the copies), so a rank never materialises the global matrix on the host.
namespace {

thread_local std::string g_io_error;

constexpr uint64_t kUotpHeader = 40;

struct UotpHeader {
  uint64_t m = 0, n = 0;
  int dtype = 0;
  double er = 0.0, ep = 0.0;
  uint64_t elem = 4;
};

int io_fail(const std::string& msg) {
  g_io_error = msg;
  return UOT_IO_ERROR;
}

uint64_t get_le(const unsigned char* p, int bytes) {
  uint64_t v = 0;
  for (int k = bytes - 1; k >= 0; --k) v = (v << 8) | p[k];
  return v;
}
void put_le(unsigned char* p, uint64_t v, int bytes) {
  for (int k = 0; k < bytes; ++k) p[k] = static_cast<unsigned char>(v >> (8 * k));
}

// read_problem's checks in its order (problem_io.cpp:106-135); little-endian host.
int read_uotp_header(int fd, const char* path, UotpHeader* h) {
  struct stat st;
  if (fstat(fd, &st) != 0) return io_fail(std::string("read_problem: cannot open ") + path);
  const uint64_t size = static_cast<uint64_t>(st.st_size);
  if (size < kUotpHeader) return io_fail("read_problem: truncated header");
  unsigned char b[kUotpHeader];
  if (pread(fd, b, kUotpHeader, 0) != static_cast<ssize_t>(kUotpHeader))
    return io_fail(std::string("read_problem: short read from ") + path);
  if (std::memcmp(b, "UOTP", 4) != 0) return io_fail("read_problem: bad magic");
  const uint64_t version = get_le(b + 4, 2);
  if (version != 1) return io_fail("read_problem: unsupported version " + std::to_string(version));
  const uint64_t dtype = get_le(b + 6, 2);
  if (dtype != 1 && dtype != 2) return io_fail("read_problem: unknown dtype code " + std::to_string(dtype));
  h->m = get_le(b + 8, 8);
  h->n = get_le(b + 16, 8);
  if (h->m < 1 || h->n < 1) return io_fail("read_problem: matrix must be at least 1x1");
  uint64_t er = get_le(b + 24, 8), ep = get_le(b + 32, 8);
  std::memcpy(&h->er, &er, 8);
  std::memcpy(&h->ep, &ep, 8);
  h->dtype = static_cast<int>(dtype);
  h->elem = dtype == 1 ? 4 : 8;
  const unsigned __int128 expected = static_cast<unsigned __int128>(kUotpHeader) +
                                     static_cast<unsigned __int128>(h->m) * h->n * h->elem +
                                     static_cast<unsigned __int128>(8) * (h->m + h->n);
  if (static_cast<unsigned __int128>(size) != expected)
    return io_fail("read_problem: payload size does not match header extents");
  return UOT_OK;
}

bool pread_all(int fd, void* buf, uint64_t bytes, uint64_t off) {
  auto* p = static_cast<unsigned char*>(buf);
  while (bytes) {
    const ssize_t r = pread(fd, p, std::min<uint64_t>(bytes, 1ull << 30), static_cast<off_t>(off));
    if (r <= 0) return false;
    p += r;
    off += static_cast<uint64_t>(r);
    bytes -= static_cast<uint64_t>(r);
  }
  return true;
}
bool pwrite_all(int fd, const void* buf, uint64_t bytes, uint64_t off) {
  auto* p = static_cast<const unsigned char*>(buf);
  while (bytes) {
    const ssize_t r = pwrite(fd, p, std::min<uint64_t>(bytes, 1ull << 30), static_cast<off_t>(off));
    if (r <= 0) return false;
    p += r;
    off += static_cast<uint64_t>(r);
    bytes -= static_cast<uint64_t>(r);
  }
  return true;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// Two page-locked staging buffers of whole rows: file <-> HBM, overlapped.
struct Staging {
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  uint64_t rows_per = 0;
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
  int init(uot_ctx* ctx) {
    const uint64_t row_bytes = ctx->cols * ctx->esz;
    rows_per = std::max<uint64_t>(1, (64ull << 20) / row_bytes);
    rows_per = std::min<uint64_t>(rows_per, ctx->rows);
    for (int i = 0; i < 2; ++i) {
      CK(cudaMallocHost(&buf[i], rows_per * row_bytes));
      CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    return UOT_OK;
  }
};

}  // namespace

extern "C" {

const char* uot_last_io_error(void) { return g_io_error.c_str(); }

int uot_problem_file_info(const char* path, uint64_t* m, uint64_t* n, int* dtype, double* er, double* ep) {
  if (!path) return UOT_INVALID_PARAMETER;
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return io_fail(std::string("read_problem: cannot open ") + path);
  UotpHeader h;
  const int rc = read_uotp_header(f.fd, path, &h);
  if (rc) return rc;
  if (m) *m = h.m;
  if (n) *n = h.n;
  if (dtype) *dtype = h.dtype;
  if (er) *er = h.er;
  if (ep) *ep = h.ep;
  return UOT_OK;
}

int uot_load_problem_file(uot_ctx* ctx, const char* path) {
  if (!ctx || !path) return UOT_INVALID_PARAMETER;
  CK(cudaSetDevice(ctx->device));
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return ctx->fail(UOT_IO_ERROR, "read_problem: cannot open %s", path);
  UotpHeader h;
  if (read_uotp_header(f.fd, path, &h)) return ctx->fail(UOT_IO_ERROR, "%s", g_io_error.c_str());
  if (h.dtype != ctx->dtype)
    return ctx->fail(UOT_INVALID_PARAMETER, "%s holds a Problem<%s>, the session a Problem<%s>", path,
                     h.dtype == UOT_F64 ? "double" : "float", ctx->dtype == UOT_F64 ? "double" : "float");
  if (h.m != ctx->global_rows || h.n != ctx->cols)
    return ctx->fail(UOT_INVALID_PARAMETER, "%s is %llux%llu, the session expects %llux%llu", path,
                     (unsigned long long)h.m, (unsigned long long)h.n, (unsigned long long)ctx->global_rows,
                     (unsigned long long)ctx->cols);
  const uint64_t mat_off = kUotpHeader, rpd_off = mat_off + h.m * h.n * h.elem, cpd_off = rpd_off + 8 * h.m;
  std::vector<double> rpd(ctx->rows), cpd(ctx->cols);
  if (!pread_all(f.fd, rpd.data(), 8 * ctx->rows, rpd_off + 8 * ctx->row_offset) ||
      !pread_all(f.fd, cpd.data(), 8 * ctx->cols, cpd_off))
    return ctx->fail(UOT_IO_ERROR, "read_problem: short read from %s", path);
  int rc = check_marginals(ctx, rpd.data(), cpd.data(), h.er, h.ep);
  if (rc) return rc;
  ctx->er = h.er;
  ctx->ep = h.ep;
  ctx->have_problem = false;
  Staging sg;
  if ((rc = sg.init(ctx))) return rc;
  const uint64_t row_bytes = ctx->cols * ctx->esz;
  for (uint64_t r0 = 0, k = 0; r0 < ctx->rows; r0 += sg.rows_per, ++k) {
    const uint64_t nr = std::min<uint64_t>(sg.rows_per, ctx->rows - r0);
    const int i = static_cast<int>(k & 1);
    CK(cudaEventSynchronize(sg.ev[i]));  // the copy out of this buffer two chunks ago is done
    if (!pread_all(f.fd, sg.buf[i], nr * row_bytes, mat_off + (ctx->row_offset + r0) * row_bytes))
      return ctx->fail(UOT_IO_ERROR, "read_problem: short read from %s", path);
    CK(cudaMemcpy2DAsync(static_cast<char*>(ctx->P) + r0 * ctx->pitch * ctx->esz, ctx->pitch * ctx->esz, sg.buf[i],
                         row_bytes, row_bytes, nr, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaEventRecord(sg.ev[i], ctx->stream));
  }
  CK(cudaMemcpyAsync(ctx->rpd, rpd.data(), ctx->rows * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->cpd, cpd.data(), ctx->cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if ((rc = reset_state(ctx))) return rc;
  if ((rc = after_matrix_upload(ctx))) return rc;  // require_valid's matrix check (problem.hpp:64-98)
  ctx->have_problem = true;
  return UOT_OK;
}

int uot_save_problem_file(uot_ctx* ctx, const char* path) {
  if (!ctx || !path) return UOT_INVALID_PARAMETER;
  if (!ctx->have_problem) return ctx->fail(UOT_INVALID_PARAMETER, "no problem set");
  CK(cudaSetDevice(ctx->device));
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT, 0644);  // every rank opens; no truncation races
  if (f.fd < 0) return ctx->fail(UOT_IO_ERROR, "write_problem: cannot open %s", path);
  const uint64_t m = ctx->global_rows, n = ctx->cols;
  const uint64_t mat_off = kUotpHeader, rpd_off = mat_off + m * n * ctx->esz, cpd_off = rpd_off + 8 * m;
  if (ftruncate(f.fd, static_cast<off_t>(cpd_off + 8 * n)) != 0)
    return ctx->fail(UOT_IO_ERROR, "write_problem: cannot size %s", path);
  if (ctx->rank == 0) {
    unsigned char b[kUotpHeader];
    std::memcpy(b, "UOTP", 4);
    put_le(b + 4, 1, 2);
    put_le(b + 6, static_cast<uint64_t>(ctx->dtype), 2);
    put_le(b + 8, m, 8);
    put_le(b + 16, n, 8);
    uint64_t er, ep;
    std::memcpy(&er, &ctx->er, 8);
    std::memcpy(&ep, &ctx->ep, 8);
    put_le(b + 24, er, 8);
    put_le(b + 32, ep, 8);
    std::vector<double> cpd(n);
    CK(cudaMemcpyAsync(cpd.data(), ctx->cpd, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (!pwrite_all(f.fd, b, kUotpHeader, 0) || !pwrite_all(f.fd, cpd.data(), 8 * n, cpd_off))
      return ctx->fail(UOT_IO_ERROR, "write_problem: short write to %s", path);
  }
  std::vector<double> rpd(ctx->rows);
  CK(cudaMemcpyAsync(rpd.data(), ctx->rpd, ctx->rows * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  Staging sg;
  int rc = sg.init(ctx);
  if (rc) return rc;
  const uint64_t row_bytes = n * ctx->esz;
  uint64_t pend_r0[2] = {0, 0}, pend_nr[2] = {0, 0};
  auto flush = [&](int i) -> bool {
    if (!pend_nr[i]) return true;
    if (cudaEventSynchronize(sg.ev[i]) != cudaSuccess) return false;
    const bool ok = pwrite_all(f.fd, sg.buf[i], pend_nr[i] * row_bytes, mat_off + (ctx->row_offset + pend_r0[i]) * row_bytes);
    pend_nr[i] = 0;
    return ok;
  };
  for (uint64_t r0 = 0, k = 0; r0 < ctx->rows; r0 += sg.rows_per, ++k) {
    const uint64_t nr = std::min<uint64_t>(sg.rows_per, ctx->rows - r0);
    const int i = static_cast<int>(k & 1);
    if (!flush(i)) return ctx->fail(UOT_IO_ERROR, "write_problem: short write to %s", path);
    CK(cudaMemcpy2DAsync(sg.buf[i], row_bytes, static_cast<const char*>(ctx->P) + r0 * ctx->pitch * ctx->esz,
                         ctx->pitch * ctx->esz, row_bytes, nr, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaEventRecord(sg.ev[i], ctx->stream));
    pend_r0[i] = r0;
    pend_nr[i] = nr;
  }
  if (!flush(0) || !flush(1)) return ctx->fail(UOT_IO_ERROR, "write_problem: short write to %s", path);
  CK(cudaStreamSynchronize(ctx->stream));
  if (!pwrite_all(f.fd, rpd.data(), 8 * ctx->rows, rpd_off + 8 * ctx->row_offset))
    return ctx->fail(UOT_IO_ERROR, "write_problem: short write to %s", path);
  return UOT_OK;
}

}  // extern "C"

#define CKC(c, expr)                                          \
  do {                                                        \
    const int _rc = (c)->cuda((expr), #expr);                 \
    if (_rc != UOT_OK) return _rc;                            \
  } while (0)

// ---------------------------------------------- single-process rank groups --
// The reference's distributed_solve(p, tol, max_iter, ranks | RankPartition)
// runs every rank in ONE process (distributed.hpp:52-136). A group is that call
// on the GPU: rank r is a peer session on devices[r] (devices may repeat), the
// exchange regions are mapped into each other directly — one address space,
// device pointers plus peer access, no IPC — and every collective step is
// enqueued phase by phase: [sweep, stage 1] on every rank's stream, an event
// per rank, then each stream waits for all ranks' events before its stage 2.
// Stage 2 therefore never waits on a rank whose kernels are queued behind it
// (ranks sharing a GPU cannot deadlock), and the result is the same ascending-
// rank exchange as the multi-process path (finalize.cuh, allreduce.cpp:6-15).
namespace {

int group_check(uot_ctx* const* ctxs, int n) {
  if (!ctxs || n < 1) return UOT_INVALID_PARAMETER;
  for (int r = 0; r < n; ++r) {
    uot_ctx* c = ctxs[r];
    if (!c) return UOT_INVALID_PARAMETER;
    if (c->nranks != n || c->rank != r || (n > 1 && !c->group_local) || c->group_id != ctxs[0]->group_id)
      return c->fail(UOT_INVALID_PARAMETER, "not rank %d of the %d-rank session group of rank 0", r, n);
  }
  return UOT_OK;
}

// One collective step of every rank: [sweep,] stage 1 | events | stage 2.
template <int MODE>
int group_step(uot_ctx* const* c, int n, bool sweep, bool seed) {
  int rc;
  for (int r = 0; r < n; ++r) {
    CKC(c[r], cudaSetDevice(c[r]->device));
    if (sweep && (rc = launch_sweep(c[r], seed))) return rc;
    if (n == 1) {
      if ((rc = launch_finalize_single<MODE>(c[r]))) return rc;
      continue;
    }
    finalize_kernel<MODE, true, false, kXchPeer>
        <<<finalize_blocks(c[r]->pitch), kFinThreads, 0, c[r]->stream>>>(fin_args(c[r]));
    c[r]->launches++;
    CKC(c[r], cudaGetLastError());
    CKC(c[r], cudaEventRecord(c[r]->xev, c[r]->stream));
  }
  if (n == 1) return UOT_OK;
  for (int r = 0; r < n; ++r) {
    CKC(c[r], cudaSetDevice(c[r]->device));
    for (int q = 0; q < n; ++q)
      if (q != r) CKC(c[r], cudaStreamWaitEvent(c[r]->stream, c[q]->xev, 0));
    finalize_kernel<MODE, false, true, kXchPeer>
        <<<finalize_blocks(c[r]->pitch), kFinThreads, 0, c[r]->stream>>>(fin_args(c[r]));
    c[r]->launches++;
    CKC(c[r], cudaGetLastError());
  }
  return UOT_OK;
}

}  // namespace

extern "C" {

int uot_create_group(uot_ctx** out, uint64_t global_rows, uint64_t cols, int dtype, const int* devices,
                     int nranks, const uint64_t* bounds) {
  if (!out || nranks < 1) return UOT_INVALID_PARAMETER;
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    ndev = 1;  // rank 0's session reports the CUDA error
  }
  std::vector<int> dev(nranks);
  for (int r = 0; r < nranks; ++r) dev[r] = devices ? devices[r] : r % ndev;
  int rc = UOT_OK;
  for (int r = 0; r < nranks && rc == UOT_OK; ++r) rc = create_peer_rank(&out[r], global_rows, cols, dtype, dev[r], r, nranks, bounds);
  if (rc) return rc;  // out[r] (if set) carries the message; the caller destroys every non-null rank
  if (nranks == 1) return UOT_OK;
  // peer access between every pair of distinct devices (NVLink / NVSwitch)
  for (int a = 0; a < nranks; ++a)
    for (int b = 0; b < nranks; ++b) {
      if (dev[a] == dev[b]) continue;
      int can = 0;
      CKC(out[a], cudaDeviceCanAccessPeer(&can, dev[a], dev[b]));
      if (!can) return out[a]->fail(UOT_CUDA_ERROR, "device %d cannot access device %d (peer access)", dev[a], dev[b]);
      CKC(out[a], cudaSetDevice(dev[a]));
      const cudaError_t e = cudaDeviceEnablePeerAccess(dev[b], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return out[a]->fail(UOT_CUDA_ERROR, "cudaDeviceEnablePeerAccess(%d -> %d): %s", dev[a], dev[b],
                            cudaGetErrorString(e));
      cudaGetLastError();  // (clear "already enabled")
    }
  static std::atomic<uint64_t> next_group{1};
  const uint64_t gid = next_group.fetch_add(1);
  for (int r = 0; r < nranks; ++r) {
    uot_ctx* c = out[r];
    c->group_id = gid;
    CKC(c, cudaSetDevice(c->device));
    c->peer_ptrs.assign(nranks, nullptr);
    for (int q = 0; q < nranks; ++q) c->peer_ptrs[q] = out[q]->region;
    CKC(c, cudaMemcpy(c->d_peers, c->peer_ptrs.data(), sizeof(unsigned char*) * nranks, cudaMemcpyHostToDevice));
    CKC(c, cudaEventCreateWithFlags(&c->xev, cudaEventDisableTiming));
    c->group_local = true;
    c->connected = true;
  }
  return UOT_OK;
}

int uot_group_init_col_sums(uot_ctx* const* ctxs, int nranks) {
  int rc = group_check(ctxs, nranks);
  if (rc) return rc;
  for (int r = 0; r < nranks; ++r) {
    if (!ctxs[r]->have_problem) return ctxs[r]->fail(UOT_INVALID_PARAMETER, "no problem set");
    CKC(ctxs[r], cudaSetDevice(ctxs[r]->device));
    if ((rc = reset_state(ctxs[r]))) return rc;
  }
  if ((rc = group_step<kFinSeed>(ctxs, nranks, true, true))) return rc;
  for (int r = 0; r < nranks; ++r) {
    CKC(ctxs[r], cudaSetDevice(ctxs[r]->device));
    if ((rc = sync_ctl(ctxs[r]))) return rc;
    ctxs[r]->seeded = true;
  }
  return UOT_OK;
}

int uot_group_iterate(uot_ctx* const* ctxs, int nranks, uint64_t k, double tol, uint64_t* iterations,
                      double* final_error, int* converged) {
  int rc = group_check(ctxs, nranks);
  if (rc) return rc;
  std::vector<uint64_t> before(nranks);
  for (int r = 0; r < nranks; ++r) {
    uot_ctx* c = ctxs[r];
    if (!c->have_problem) return c->fail(UOT_INVALID_PARAMETER, "no problem set");
    if (!c->seeded) return c->fail(UOT_INVALID_PARAMETER, "carried column sums missing (call init_col_sums)");
    if (!(tol > 0.0)) return c->fail(UOT_INVALID_PARAMETER, "tol must be positive");
    if (k < 1) return c->fail(UOT_INVALID_PARAMETER, "max_iter must be at least 1");
    if (c->variant != UOT_VARIANT_FUSED) return c->fail(UOT_INVALID_PARAMETER, "groups run the fused schedule");
    before[r] = c->h_ctl->iter;
    CKC(c, cudaSetDevice(c->device));
    begin_iterate_kernel<<<1, 1, 0, c->stream>>>(c->ctl, tol);
    c->launches++;
    CKC(c, cudaGetLastError());
  }
  for (uint64_t i = 0; i < k; ++i)
    if ((rc = group_step<kFinIter>(ctxs, nranks, true, false))) return rc;
  for (int r = 0; r < nranks; ++r) {
    CKC(ctxs[r], cudaSetDevice(ctxs[r]->device));
    if ((rc = sync_ctl(ctxs[r]))) return rc;
  }
  for (int r = 0; r < nranks; ++r)
    if ((rc = status_of(ctxs[r]))) return rc;
  const Control& h0 = *ctxs[0]->h_ctl;
  for (int r = 1; r < nranks; ++r) {  // every rank derives the same factors and the same stop decision
    const Control& h = *ctxs[r]->h_ctl;
    if (h.iter - before[r] != h0.iter - before[0] || h.converged != h0.converged)
      return ctxs[r]->fail(UOT_CUDA_ERROR, "rank %d stopped after %llu iterations, rank 0 after %llu", r,
                           (unsigned long long)(h.iter - before[r]), (unsigned long long)(h0.iter - before[0]));
  }
  if (iterations) *iterations = h0.iter - before[0];
  if (final_error) *final_error = h0.last_error;
  if (converged) *converged = h0.converged;
  return UOT_OK;
}

}  // extern "C"
