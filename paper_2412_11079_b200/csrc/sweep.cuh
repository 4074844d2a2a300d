// sweep.cuh — the fused MAP-UOT iteration as ONE sm_100a streaming kernel.
//
// Reference semantics (paths under /root/reference/proj/core):
//   detail::fused_row_pass  include/uot/fused.hpp:119-144
//     sweep 1: x <- f32(f64(x) * beta_j); s += f64(x)        (125-131)
//     alpha_i = rescale_factor(rpd_i, s, fi)                 (133; src/scaling.cpp:15-22)
//     sweep 2: x <- f32(f64(x) * alpha_i); next_j += f64(x)  (135-142)
//   init_col_sums (the seed)  include/uot/fused.hpp:96-110
//   ordered partial reduction include/uot/fused.hpp:242-248 -> finalize.cuh
//
// B200 design:
//   * P is row-major [rows][pitch] fp32 in HBM; each row is cut into G column
//     slices of `slice` floats (G = ceil(cols/8192)). A "group" of G CTAs owns a
//     contiguous, balanced block of rows (plan.cpp:11-21 rule); CTA g of the
//     group owns slice g of every row in the block. grid = groups * G <= #SMs,
//     one CTA per SM, persistent over the block.
//   * Warp roles. A producer warp streams batches (B rows of the CTA's slice)
//     through a ring of NBUF shared-memory slots with 1-D bulk copies (TMA
//     engine, UBLKCP) signalled on mbarriers and bulk-stores finished batches
//     back. Both sweeps run in place in shared memory, so P is read from and
//     written to HBM exactly once per iteration. NF factor warps turn row sums
//     into row factors. NW compute warps do the arithmetic.
//   * Compute warps never meet a CTA-wide barrier: they wait only for data
//     (full) and factors (alpha_rdy) and hand work on through mbarriers (done1:
//     row partials written; done2: sweep 2 finished).
//     Slices of V >= 2 float4 per thread, batches of <= 2 rows: SPLIT roles —
//     half the compute warps run sweep 1 + the row partials of every batch as
//     soon as it lands (paced by the ring only), the other half sweep 2 + the
//     column partials once the batch's factors are published; each thread
//     covers 2V chunks, each warp waits on one barrier per batch (measured -2%
//     at 32768^2, 131072x32768 and 262144x4096, -4% at 8192^2 against both
//     sweeps in every warp).
//     Other slices: step s runs sweep 1 of batch s, then sweep 2 of batch
//     s-LA-1, then the row reduction of batch s, in every compute warp.
//   * Per-column state of the owning thread: beta_j (f64, registers or TMEM)
//     and the column partial next_j (f64, registers). Thread t owns float4
//     chunks t, t+NT, ... of the slice (conflict-free 128-bit smem access).
//   * Row sums: thread partial -> warp xor-tree -> per-warp smem -> factor lane
//     sums the NW warp partials in warp order. With G > 1 the G CTA partials of
//     a row are exchanged through L2 as 128-bit single-copy-atomic {value, tag}
//     records (no fences), summed in ascending g, so every CTA of the group
//     derives the bit-identical alpha_i. No float atomics: deterministic.
//   * Arithmetic is exactly the reference's: f64 products rounded once to fp32
//     (F2F.F32.F64), f64 sums of the stored fp32 values (see ScreenBounds).
#pragma once
#include <cstdint>
#include <type_traits>

#include "ptx.cuh"
#include "uot_device.cuh"

namespace uotk {

struct SweepArgs {
  void* P;                    // [rows][pitch] fp32 (or fp64: Problem<double>), device layout
  const double* beta2;        // [2][pitch] column factors; beta(t) lives in slot t&1
  const double* rpd;          // [rows] row marginals
  double* alpha;              // [rows] row factors (output)
  double* partials;           // [groups][pitch] column partials (output)
  double* cta_err;            // [grid][kErrSlots] max|alpha-1| seen by each CTA's factor warps (output)
  ulonglong2* xrec;           // [grid][kRing] exchanged {partial bits, tag} (G > 1)
  Control* ctl;
  unsigned long long rows;    // local rows
  unsigned int pitch;         // floats per device row (= G * slice)
  unsigned int slice;         // floats per CTA column slice (multiple of 4)
  unsigned int G;             // CTAs per row group
  unsigned int groups;        // row groups
  unsigned int B;             // rows per pipeline batch (<= BM; 1 when G > 1)
  unsigned int buf_stride;    // bytes per smem ring slot (128-aligned, >= B*slice*4)
  int evict_first;            // stream P past L2 (problem larger than L2)
  int smid_map;               // CTA slot = %smid (the grid covers every SM exactly once)
  const unsigned* slot_of_sm; // [#SMs] CTA slot of each SM (class-grouped row groups), or nullptr
  const unsigned long long* gbounds;  // [groups+1] static row block of each group, or nullptr (balanced)
  unsigned* dbg;              // [grid][kDbg] {smid, batches, start, end ns} of the last sweep (schedule statistics)
  int dyn;                    // batches handed out by a global counter (else a static row block)
  unsigned keep;              // static blocks: a CTA stores its last `keep` batches L2-resident (evict_last)
                              // and walks its block in alternating directions, so the next sweep starts on them
  ulonglong2* mail;           // [groups][kMail] {first row, tag}: the group leader's batch picks (dyn, G > 1)
  double fi;
};

// Optional wait timers (build with -DUOT_TRACE): clock64 cycles spent in the
// waits only (6 registers, so the build runs at close to full speed), summed
// over CTAs into uot_trace[] and read back with uot_trace_read(): 0 factor wait
// done1, 2 exchange poll, 3 pow+arrive, 4 producer wait done2, 16 compute wait
// full, 19 compute wait alpha; 8/9/21 role totals.
#ifdef UOT_TRACE
__device__ unsigned long long uot_trace[32];
__host__ __device__ constexpr int tr_slot(int id) {
  return id == 0 ? 0 : id == 2 ? 1 : id == 3 ? 2 : id == 4 ? 3 : id == 16 ? 4 : id == 19 ? 5 : -1;
}
#define TR_DECL unsigned long long tr_t0 = 0, tr_acc[6] = {0, 0, 0, 0, 0, 0}; (void)tr_t0;
#define TR_BEGIN() tr_t0 = clock64()
#define TR_END(id)                                                  \
  do {                                                              \
    if (tr_slot(id) >= 0) tr_acc[tr_slot(id)] += clock64() - tr_t0; \
  } while (0)
#define TR_FLUSH(lo, hi)           \
  for (int i_ = lo; i_ < hi; ++i_) \
    if (tr_slot(i_) >= 0) atomicAdd(&uot_trace[i_], tr_acc[tr_slot(i_) < 0 ? 0 : tr_slot(i_)])
#else
#define TR_DECL
#define TR_BEGIN()
#define TR_END(id)
#define TR_FLUSH(lo, hi)
#endif

constexpr int kRing = 16;  // exchange records per CTA (> how far a CTA's factor warps can run ahead of a peer's)
constexpr int kDbg = 4;    // schedule statistics per CTA: SM id, row batches, producer start / end (globaltimer ns, low 32 bits)
constexpr int kQ = 4;      // ring depth of row partials / factors handed between roles (>= LA + 2)
constexpr int kQMax = 12;  // smem reserved for the row-partial / factor rings (split roles: > NBUF, multiple of NF)
constexpr int kMail = 32;  // batch picks a group leader publishes ahead of its followers
constexpr unsigned long long kNoRow = ~0ull;  // ring slot sentinel: no batch left

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // xor tree: every lane holds the bit-identical total (fp add commutes)
}

// Row-sum exchange of a G-CTA row group (G > 1): publish this CTA's partial of
// the row as a 128-bit single-copy-atomic {value, tag} record in L2 (no
// fences), then gather the G records of the row — one lane per record, 32 at a
// time, spinning on L2 (any back-off costs more than the polls) — and add them
// in ascending g: identical bits on every CTA of the group. Whole warp calls.
__device__ __forceinline__ double exchange_row_sum(ulonglong2* xrec, unsigned cta, unsigned group, unsigned G,
                                                   unsigned slot, unsigned long long tag, double t, Control* ctl) {
  const unsigned lane = threadIdx.x & 31;
  if (lane == 0)
    st_relaxed_b128(&xrec[static_cast<size_t>(cta) * kRing + slot],
                    static_cast<unsigned long long>(__double_as_longlong(t)), tag);
  double tot = 0.0;
  for (unsigned g0 = 0; g0 < G; g0 += 32) {
    double v = 0.0;
    // every lane polls, its own CTA's record included (measured: skipping the
    // own record and using t directly is 1.5% slower at 32768^2)
    if (g0 + lane < G) {
      const ulonglong2* rec = &xrec[static_cast<size_t>(group * G + g0 + lane) * kRing + slot];
      unsigned long long lo, hi;
      ld_relaxed_b128(rec, lo, hi);
      if (hi != tag) {
        const unsigned long long t0 = globaltimer_ns();
        unsigned n = 0;
        do {
          ld_relaxed_b128(rec, lo, hi);
          if (hi != tag && (++n & 255u) == 0 && globaltimer_ns() - t0 > kExchangeTimeoutNs) {
#ifdef UOT_DEBUG
            printf("xchg timeout cta %u group %u slot %u tag %llx seen %llx (rec of cta %u)\n", cta, group, slot, tag, hi,
                   group * G + g0 + lane);
#endif
            atomicOr(&ctl->status, kStatusExchangeTimeout);
            break;
          }
        } while (hi != tag);
      }
      v = __longlong_as_double(static_cast<long long>(lo));
    }
    const unsigned n = min(32u, G - g0);
    for (unsigned k = 0; k < n; ++k) tot += __shfl_sync(0xffffffffu, v, k);
  }
  return tot;
}

// ------------------------------------------------------ per-row sweep bodies --
// A thread owns float4 chunks q = tid + k*NT (k < V) of the slice. FULL: every
// chunk exists (slice == 4*NT*V); otherwise missing chunks carry 1.0f through
// the arithmetic and are never stored or summed.
//
// Exactness. f32 -> f64 is two integer ops (fastd) for positive normal floats
// (hardware F2F.F64.F32 runs on the 16/clk/SM conversion pipe, which caps the
// sweep near the HBM rate: profiles/r01_conv_microbench.txt). Each group of x0
// values is screened with one VIADDMNMX per value against a per-thread window
// (ScreenBounds) that certifies x0 positive normal and x1 = f32(f64(x0)*beta_j)
// inside [FLT_MIN*2^20, FLT_MAX*2^-20]; otherwise the group takes exact hardware
// conversions. A row whose factor alpha lies in [2^-20, 2^20] then maps every
// certified x1 to a positive normal x2 = f32(f64(x1)*alpha), so sweep 2 widens
// x1 and x2 with fastd and no screen at all; other rows (and rows with an
// uncertified group) take the hardware conversions. f64 -> f32 is one
// F2F.F32.F64 (RN), the reference's T(double).

__device__ __forceinline__ uint32_t nn_max(uint32_t m, float x) {
  return max(m, __float_as_uint(x) - 0x800000u);  // >= 0x7f000000 <=> not positive normal
}
__device__ __forceinline__ bool nn_ok(uint32_t m) { return m < 0x7f000000u; }
__device__ __forceinline__ double fastd(float x) {
  const uint32_t u = __float_as_uint(x);
  return __hiloint2double(static_cast<int>((u >> 3) + 0x38000000u), static_cast<int>(u << 29));
}
__device__ __forceinline__ float& comp(float4& v, int e) {
  return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}

// Chunks are processed in groups of KG float4 (8 values for KG = 2): one screen
// and one branch per group keeps the fast path branch-light while bounding the
// live registers under the 96-register cap of a 19-warp CTA.
template <int V>
struct ChunkGroup {
  static constexpr int KG = (V <= 2 || V % 2 != 0) ? V : 2;
  static_assert(V % KG == 0, "V must be a multiple of the chunk group");
};

// Screen window of a thread: x0 passes iff lo <= x0 <= hi as floats, with
// lo = max(FLT_MIN, FLT_MIN*M/beta_min), hi = min(FLT_MAX, FLT_MAX/(M*beta_max))
// rounded inward over the thread's beta_j (M = kAlphaMargin): then x0*beta_j
// lies in [FLT_MIN*M, FLT_MAX/M] exactly, and both rounding steps keep x1 there
// (the bounds are representable), so x1*alpha stays positive normal for every
// alpha in [1/M, M].
constexpr double kAlphaMargin = 0x1p20;
struct ScreenBounds {
  uint32_t lo, span;  // bits(lo), bits(hi) - bits(lo)
};
__device__ __forceinline__ ScreenBounds screen_bounds(const double* beta, int n) {
  // padding columns carry beta = 0 and x = 0: they fail any window, so skip them
  double bmin = 1e308, bmax = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) {
    if (beta[i] > 0.0) {
      bmin = fmin(bmin, beta[i]);
      bmax = fmax(bmax, beta[i]);
    }
  }
  if (!(bmax > 0.0)) bmin = bmax = 1.0;
  const double tiny = 1.1754943508222875e-38, big = 3.4028234663852886e38;  // FLT_MIN, FLT_MAX
  const float lo = __double2float_ru(fmax(tiny, tiny * kAlphaMargin / bmin * (1.0 + 0x1p-40)));
  const float hi = __double2float_rd(fmin(big, big / (kAlphaMargin * bmax) * (1.0 - 0x1p-40)));
  ScreenBounds b;
  b.lo = __float_as_uint(lo);
  b.span = (bmax < 1e300 && lo <= hi) ? __float_as_uint(hi) - __float_as_uint(lo) : 0u;
  if (b.span == 0u) b.lo = 0xffffffffu;  // empty window: every group takes the exact path
  return b;
}
__device__ __forceinline__ uint32_t sc_max(uint32_t m, float x, uint32_t lo) {
  return max(m, __float_as_uint(x) - lo);  // wraps for x < lo: fails the window test
}

// Sweep 1 of one chunk group (fused.hpp:125-131): x <- f32(f64(x)*beta_j) in
// place, t[e] = sum of f64(x); `bad` when the group took the exact path.
template <int NT, int KG, bool FULL>
__device__ __forceinline__ void group_sweep1(float4* row, float4 (&v)[KG], uint32_t m, int g0, unsigned tid,
                                             unsigned nq, const double* beta, ScreenBounds sb, double (&t)[4],
                                             bool& bad) {
  if (m <= sb.span) {  // x0 and x1 certified positive normal: two-op widening both times
#pragma unroll
    for (int kk = 0; kk < KG; ++kk)
#pragma unroll
      for (int e = 0; e < 4; ++e) comp(v[kk], e) = d2f(fastd(comp(v[kk], e)) * beta[4 * (g0 + kk) + e]);
    const bool ok0 = FULL || tid + g0 * NT < nq;
#pragma unroll
    for (int e = 0; e < 4; ++e) t[e] = ok0 ? fastd(comp(v[0], e)) : 0.0;  // (no 0.0 + x DADD)
#pragma unroll
    for (int kk = 1; kk < KG; ++kk)
      if (FULL || tid + (g0 + kk) * NT < nq)
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e] += fastd(comp(v[kk], e));
  } else {  // exact hardware conversions for any input
    bad = true;
#pragma unroll
    for (int kk = 0; kk < KG; ++kk)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        comp(v[kk], e) = d2f(static_cast<double>(comp(v[kk], e)) * beta[4 * (g0 + kk) + e]);
    const bool ok0 = FULL || tid + g0 * NT < nq;
#pragma unroll
    for (int e = 0; e < 4; ++e) t[e] = ok0 ? static_cast<double>(comp(v[0], e)) : 0.0;
#pragma unroll
    for (int kk = 1; kk < KG; ++kk)
      if (FULL || tid + (g0 + kk) * NT < nq)
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e] += static_cast<double>(comp(v[kk], e));
  }
#pragma unroll
  for (int kk = 0; kk < KG; ++kk) {
    const unsigned q = tid + (g0 + kk) * NT;
    if (FULL || q < nq) row[q] = v[kk];
  }
}

// Sweep 2 of one chunk group (fused.hpp:135-142): x <- f32(f64(x)*alpha) in
// place, next_j += f64(x). !EXACT: x1 certified by sweep 1's screen and alpha
// in [1/M, M], so x1 and x2 are positive normal (fastd both times, +1.3% over
// the hardware conversion at 32768^2); EXACT: hardware conversions.
template <int NT, int KG, bool FULL, bool EXACT>
__device__ __forceinline__ void group_sweep2(float4* row, float4 (&w)[KG], int g0, unsigned tid, unsigned nq,
                                             double al, double* acc) {
#pragma unroll
  for (int kk = 0; kk < KG; ++kk)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      comp(w[kk], e) = d2f((EXACT ? static_cast<double>(comp(w[kk], e)) : fastd(comp(w[kk], e))) * al);
#pragma unroll
  for (int kk = 0; kk < KG; ++kk) {
    const unsigned q = tid + (g0 + kk) * NT;
    if (FULL || q < nq) {
      row[q] = w[kk];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        acc[4 * (g0 + kk) + e] += EXACT ? static_cast<double>(comp(w[kk], e)) : fastd(comp(w[kk], e));
    }
  }
}

template <int NT, int KG, bool FULL>
__device__ __forceinline__ void load_group(const float4* row, float4 (&v)[KG], int g0, unsigned tid, unsigned nq) {
#pragma unroll
  for (int kk = 0; kk < KG; ++kk) {
    const unsigned q = tid + (g0 + kk) * NT;
    v[kk] = (FULL || q < nq) ? row[q] : make_float4(1.f, 1.f, 1.f, 1.f);
  }
}

template <int KG>
__device__ __forceinline__ uint32_t screen_group(float4 (&v)[KG], uint32_t lo) {
  uint32_t m = 0;
#pragma unroll
  for (int kk = 0; kk < KG; ++kk)
#pragma unroll
    for (int e = 0; e < 4; ++e) m = sc_max(m, comp(v[kk], e), lo);
  return m;
}

// Sweep 1 of this thread's part of one row; returns the f64 row partial.
template <int NT, int V, bool FULL>
__device__ __forceinline__ double row_sweep1(float4* row, unsigned tid, unsigned nq, const double* beta,
                                             ScreenBounds sb, bool& bad) {
  constexpr int KG = ChunkGroup<V>::KG;
  double s[4];
#pragma unroll
  for (int g0 = 0; g0 < V; g0 += KG) {
    float4 v[KG];
    load_group<NT, KG, FULL>(row, v, g0, tid, nq);
    const uint32_t m = screen_group<KG>(v, sb.lo);
    double t[4];
    group_sweep1<NT, KG, FULL>(row, v, m, g0, tid, nq, beta, sb, t, bad);
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = g0 == 0 ? t[e] : s[e] + t[e];
  }
  return (s[0] + s[1]) + (s[2] + s[3]);
}

// ---- column factors parked in TMEM (TB builds) ----------------------------
// A compute thread's 4V column factors (f64, two 32-bit TMEM columns each) sit
// in its own TMEM lane: warp w owns lanes 32*(w%4).. and 8V columns from
// 8V*(w/4). Sweep 1 loads a chunk group's factors right before use, which frees
// the 8V registers the factors otherwise occupy for the whole sweep.
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc_cols(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc_cols(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tmem_st_chunk(uint32_t taddr, const double* b) {  // 4 doubles, .x8
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(__double2loint(b[0])), "r"(__double2hiint(b[0])), "r"(__double2loint(b[1])),
               "r"(__double2hiint(b[1])), "r"(__double2loint(b[2])), "r"(__double2hiint(b[2])),
               "r"(__double2loint(b[3])), "r"(__double2hiint(b[3]))
               : "memory");
}
__device__ __forceinline__ void tmem_ld_chunk(uint32_t taddr, double* b) {  // 4 doubles, .x8 (no wait)
  int w[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "r"(taddr)
               : "memory");
#pragma unroll
  for (int e = 0; e < 4; ++e) b[e] = __hiloint2double(w[2 * e + 1], w[2 * e]);
}
__device__ __forceinline__ void tmem_wait_ld_() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st_() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_before_() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after_() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Sweep 1 with the factors of each chunk group loaded from TMEM (tcol: this
// thread's first factor column).
template <int NT, int V, bool FULL, int KG0 = ChunkGroup<V>::KG>
__device__ __forceinline__ double row_sweep1_tb(float4* row, unsigned tid, unsigned nq, uint32_t tcol,
                                                ScreenBounds sb, bool& bad) {
  constexpr int KG = KG0;  // (KG = 4 measured slower with both sweeps in one warp: it spills)
  double s[4];
#pragma unroll
  for (int g0 = 0; g0 < V; g0 += KG) {
    double bq[4 * V];
#pragma unroll
    for (int kk = 0; kk < KG; ++kk) tmem_ld_chunk(tcol + 8 * (g0 + kk), bq + 4 * (g0 + kk));
    float4 v[KG];
    load_group<NT, KG, FULL>(row, v, g0, tid, nq);
    const uint32_t m = screen_group<KG>(v, sb.lo);
    tmem_wait_ld_();
    double t[4];
    group_sweep1<NT, KG, FULL>(row, v, m, g0, tid, nq, bq, sb, t, bad);
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = g0 == 0 ? t[e] : s[e] + t[e];
  }
  return (s[0] + s[1]) + (s[2] + s[3]);
}

// Sweep 2 of this thread's part of one row. `exact`: one of the thread's
// chunk groups of the row took the exact path in sweep 1.
template <int NT, int V, bool FULL, int KG0 = ChunkGroup<V>::KG>
__device__ __forceinline__ void row_sweep2(float4* row, unsigned tid, unsigned nq, double al, bool exact,
                                           double* acc) {
  constexpr int KG = KG0;
  exact = exact || !(al >= 1.0 / kAlphaMargin && al <= kAlphaMargin);
#pragma unroll
  for (int g0 = 0; g0 < V; g0 += KG) {
    float4 w[KG];
    load_group<NT, KG, FULL>(row, w, g0, tid, nq);
    if (exact)
      group_sweep2<NT, KG, FULL, true>(row, w, g0, tid, nq, al, acc);
    else
      group_sweep2<NT, KG, FULL, false>(row, w, g0, tid, nq, al, acc);
  }
}

// fused.hpp:96-110 seed: next_j += f64(x) over the stored values.
template <int NT, int V, bool FULL>
__device__ __forceinline__ void row_seed(const float4* row, unsigned tid, unsigned nq, double* acc) {
  constexpr int KG = ChunkGroup<V>::KG;
#pragma unroll
  for (int g0 = 0; g0 < V; g0 += KG) {
    float4 v[KG];
    load_group<NT, KG, FULL>(row, v, g0, tid, nq);
    uint32_t m = 0;
#pragma unroll
    for (int kk = 0; kk < KG; ++kk)
#pragma unroll
      for (int e = 0; e < 4; ++e) m = nn_max(m, comp(v[kk], e));
    const bool ok = nn_ok(m);
#pragma unroll
    for (int kk = 0; kk < KG; ++kk)
      if (FULL || tid + (g0 + kk) * NT < nq)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          acc[4 * (g0 + kk) + e] += ok ? fastd(comp(v[kk], e)) : static_cast<double>(comp(v[kk], e));
  }
}

// ---- Problem<double> (Dtype::f64) bodies: fused.hpp:128-140 with T = double,
// so x1 = x0*beta_j and x2 = x1*alpha are plain f64 products (no rounding to a
// narrower type) and the sums add them directly. A thread owns double2 chunks
// q = tid + k*NT (k < V).
template <int NT, int V, bool FULL>
__device__ __forceinline__ double row_sweep1_f64(double2* row, unsigned tid, unsigned nq, const double* beta) {
  double2 v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const unsigned q = tid + k * NT;
    v[k] = (FULL || q < nq) ? row[q] : make_double2(0.0, 0.0);
  }
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const unsigned q = tid + k * NT;
    v[k].x *= beta[2 * k];
    v[k].y *= beta[2 * k + 1];
    if (FULL || q < nq) {
      row[q] = v[k];
      s0 += v[k].x;
      s1 += v[k].y;
    }
  }
  return s0 + s1;
}
template <int NT, int V, bool FULL>
__device__ __forceinline__ void row_sweep2_f64(double2* row, unsigned tid, unsigned nq, double al, double* acc) {
  double2 v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const unsigned q = tid + k * NT;
    v[k] = (FULL || q < nq) ? row[q] : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const unsigned q = tid + k * NT;
    v[k].x *= al;
    v[k].y *= al;
    if (FULL || q < nq) {
      row[q] = v[k];
      acc[2 * k] += v[k].x;
      acc[2 * k + 1] += v[k].y;
    }
  }
}
template <int NT, int V, bool FULL>
__device__ __forceinline__ void row_seed_f64(const double2* row, unsigned tid, unsigned nq, double* acc) {
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const unsigned q = tid + k * NT;
    if (FULL || q < nq) {
      const double2 v = row[q];
      acc[2 * k] += v.x;
      acc[2 * k + 1] += v.y;
    }
  }
}

// Row batches of one CTA's sweep (the producer's schedule), as {first row, rows}
// packed into 64 bits (rows in the top byte), or kNoRow once the CTA's batches
// are exhausted (pick.nb = the local batch count from then on). Static: the
// group's contiguous block [r0, r1) (balanced_blocks, plan.cpp:11-21, or the
// weighted bounds), walked backwards when `back`. Dynamic: batches of B rows
// from a global counter (ctl->batch_next), so faster SMs take more of them —
// per-SM HBM bandwidth on B200 differs by up to 2x with the GPC an SM sits in
// (tools/microbench/stream_bench.cu); with G > 1 the group leader picks and
// publishes its pick to the followers through the group's mailbox ring.
struct BatchPick {
  Control* ctl;
  ulonglong2* mail;                   // this group's [kMail] ring
  unsigned long long r0, r1, nbt, mtag, rows;
  unsigned B, G, g, nb_static;
  bool dyn, back;
  unsigned nb = 0xffffffffu;
  __device__ unsigned long long operator()(unsigned b) {
    if (b >= nb) return kNoRow;
    unsigned long long row;
    if (!dyn) {
      if (b >= nb_static) {
        row = kNoRow;
      } else if (back) {  // batch b covers [max(r0, hi - B), hi), hi = r1 - b*B (rows ascending inside)
        const unsigned long long hi = r1 - static_cast<unsigned long long>(b) * B;
        const unsigned long long lo = hi > r0 + B ? hi - B : r0;
        row = lo | ((hi - lo) << 56);
      } else {
        row = r0 + static_cast<unsigned long long>(b) * B;
        row |= min(static_cast<unsigned long long>(B), r1 - row) << 56;
      }
    } else if (G == 1 || g == 0) {
      const unsigned long long t = atomicAdd(&ctl->batch_next, 1ull);
      row = t < nbt ? t * B : kNoRow;
      if (row != kNoRow) row |= min(static_cast<unsigned long long>(B), rows - row) << 56;
      if (G > 1) st_relaxed_b128(&mail[b % kMail], row, mtag | (b + 1));
    } else {
      unsigned long long lo, hi;
      ld_relaxed_b128(&mail[b % kMail], lo, hi);
      if (hi != (mtag | (b + 1))) {
        const unsigned long long t0 = globaltimer_ns();
        unsigned n = 0;
        do {
          ld_relaxed_b128(&mail[b % kMail], lo, hi);
          if (hi != (mtag | (b + 1)) && (++n & 255u) == 0 && globaltimer_ns() - t0 > kExchangeTimeoutNs) {
            atomicOr(&ctl->status, kStatusExchangeTimeout);
            lo = kNoRow;
            break;
          }
        } while (hi != (mtag | (b + 1)));
      }
      row = lo;
    }
    if (row == kNoRow) nb = b;
    return row;
  }
};
__device__ __forceinline__ unsigned rows_of_batch(unsigned long long v) { return static_cast<unsigned>(v >> 56); }
__device__ __forceinline__ unsigned long long row_of_batch(unsigned long long v) { return v & ((1ull << 56) - 1); }

// Elements per 16-byte chunk of the storage type.
template <typename T>
constexpr int elems_per_chunk() {
  return static_cast<int>(16 / sizeof(T));
}

// Shared-memory layout shared by host sizing and the kernel.
template <int NW, int BM, int NBUF>
struct SweepSmem {
  static constexpr int kQS = BM <= 2 ? kQMax : kQ;  // ring slots reserved (split roles: batches of <= 2 rows)
  static constexpr int kRed = kQ * NW * BM > kQS * (NW / 2) * BM ? kQ * NW * BM : kQS * (NW / 2) * BM;
  static constexpr int kBars = NBUF /*full*/ + NBUF /*done2*/ + kQS /*done1*/ + kQS /*alpha_rdy*/;
  static constexpr int kDoubles = kRed /*red*/ + kQS * BM /*alpha*/ + NBUF /*first row of each slot*/ +
                                  1 /*TMEM base*/ + kQS * NW / 4 /*exact-path masks (u32, [kQS][NW/2])*/;
  static size_t bytes(unsigned buf_stride) {
    return static_cast<size_t>(NBUF) * buf_stride + kBars * 8 + kDoubles * 8;
  }
};

// NT compute threads + a producer warp + NF factor warps. V float4 chunks per
// thread per row (slice <= 4*NT*V; FULL: equality), BM max rows per batch, NBUF
// ring slots. LA: batches between sweep 1 and sweep 2 of a batch beyond the
// next one (the factor warps' latency budget). XCHG: G > 1, row sums are
// exchanged across the group. SEED: the read-only init_col_sums sweep. T: the
// storage type of P (float: Problem<float>, double: Problem<double>).
template <int NT, int V, int BM, int NBUF, int LA, bool XCHG, int NF, bool FULL, bool SEED, typename T = float,
          bool TB0 = false>
__global__ void __launch_bounds__(NT + 32 * (1 + NF), 1) sweep_kernel(const SweepArgs a) {
  constexpr int NW = NT / 32;
  constexpr bool F64 = std::is_same<T, double>::value;
  constexpr bool TB = TB0 && !F64 && !SEED && NW % 4 == 0;  // column factors in TMEM
  constexpr int kTbCols = (8 * V * (NW / 4) <= 32) ? 32 : (8 * V * (NW / 4) <= 64) ? 64 : (8 * V * (NW / 4) <= 128) ? 128 : 256;
  // Split roles: half the compute warps run sweep 1 (and the row sums) over the
  // whole slice, the other half sweep 2 (and the column sums); sweep-1 warps are
  // paced by the ring only, so the row-partial / factor rings hold QD > NBUF
  // batches (a multiple of NF: each ring slot is served by one factor warp).
  constexpr bool SPLIT = !SEED && !F64 && NW % 8 == 0 && BM <= 2 && (TB || V == 2);
  constexpr int QD = SPLIT ? (NF == 3 ? 9 : 8) : kQ;
  constexpr int NWR = SPLIT ? NW / 2 : NW;  // warps contributing row partials
  static_assert(!SPLIT || (QD > NBUF && QD % NF == 0 && QD <= SweepSmem<NW, BM, NBUF>::kQS), "split-role rings");
  constexpr int EPC = elems_per_chunk<T>();  // 4 floats or 2 doubles per 16-byte chunk
  static_assert(NF >= 1 && NF <= kErrSlots, "factor warps");
  static_assert(LA >= 1 && LA + 2 <= kQ && (!XCHG || LA >= 2), "lag (the alpha / red rings hold kQ batches)");
  static_assert(NBUF >= LA + 4, "ring too small");
  static_assert(!XCHG || BM == 1, "the exchange path moves one row per batch");

  extern __shared__ __align__(128) unsigned char smem[];
  Control* ctl = a.ctl;
  if (ctl->done) return;
  if (!SEED && ctl->beta_bad) {  // beta_from_state threw at the top of this iteration
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(&ctl->status, kStatusDegenerateBeta);
      ctl->done = 1;
    }
    return;
  }

  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NBUF * a.buf_stride);
  uint64_t* done2 = full + NBUF;
  uint64_t* done1 = done2 + NBUF;
  constexpr int kQS = SweepSmem<NW, BM, NBUF>::kQS;
  uint64_t* alpha_rdy = done1 + kQS;
  double* red = reinterpret_cast<double*>(alpha_rdy + kQS);  // [QD][NWR][BM]
  double* alpha_s = red + SweepSmem<NW, BM, NBUF>::kRed;      // [QD][BM]
  // first row of the batch in each ring slot (kNoRow: the CTA's batches are
  // exhausted), written by the producer before the slot's full barrier
  unsigned long long* srow = reinterpret_cast<unsigned long long*>(alpha_s + kQS * BM);
  uint32_t* tmem_s = reinterpret_cast<uint32_t*>(srow + NBUF);  // TMEM base (TB)
  uint32_t* xbad = tmem_s + 2;  // [QD][NWR] split roles: a sweep-1 warp took the exact path on the batch

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned G = a.G;
  // CTA slot: blockIdx, or (smid_map) the SM id, so the G CTAs of a row group
  // sit on neighbouring SMs (same TPC pair / GPC, same die).
  const unsigned cta = a.slot_of_sm ? a.slot_of_sm[smid()] : (a.smid_map ? smid() : blockIdx.x);
  const unsigned group = cta / G, g = cta % G;
  // balanced_blocks over groups (plan.cpp:11-21): first rows%groups get one more.
  // Row batches. Static: group `group` owns a contiguous block of rows
  // (balanced_blocks, plan.cpp:11-21). Dynamic: batches of B rows are handed
  // out by a global counter (ctl->batch_next), so faster SMs take more of
  // them — per-SM HBM bandwidth on B200 differs by up to 2x with the GPC an SM
  // sits in (tools/microbench/stream_bench.cu). With G > 1 the group leader
  // picks and publishes its pick to the followers through `mail`.
  const unsigned B = a.B;
  const unsigned long long base = a.rows / a.groups, rem = a.rows % a.groups;
  // static row block of the group: class-weighted bounds (topology.cuh) or balanced_blocks
  const unsigned long long r0 = a.gbounds ? a.gbounds[group] : group * base + (group < rem ? group : rem);
  const unsigned long long r1 = a.gbounds ? a.gbounds[group + 1] : r0 + base + (group < rem ? 1 : 0);
  const unsigned nb_static = static_cast<unsigned>((r1 - r0 + B - 1) / B);
  const unsigned nq = a.slice / EPC;
  const uint32_t row_bytes = a.slice * static_cast<uint32_t>(sizeof(T));
  T* gbase = static_cast<T*>(a.P) + static_cast<size_t>(g) * a.slice;

  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&done2[i], NWR);
    }
    for (int i = 0; i < QD; ++i) {
      mbar_init(&done1[i], NWR);
      mbar_init(&alpha_rdy[i], 1);
    }
    fence_mbar_init();
  }
  if (TB && warp == 0) tmem_alloc_cols<kTbCols>(tmem_s);  // compute warp 0 (warp-collective)
  if (TB) tmem_fence_before_();
  __syncthreads();
  if (TB) tmem_fence_after_();
  const uint32_t tbase = TB ? *tmem_s : 0u;

  auto slot_ptr = [&](unsigned b) -> T* {
    return reinterpret_cast<T*>(smem + (b % NBUF) * a.buf_stride);
  };
  // A slot's batch travels as {first row, rows} packed into 64 bits (rows in
  // the top byte): static blocks end inside a batch, dynamic batches at `rows`.
  auto rows_at = [](unsigned long long v) -> unsigned { return static_cast<unsigned>(v >> 56); };
  auto row_of = [](unsigned long long v) -> unsigned long long { return v & ((1ull << 56) - 1); };
  TR_DECL

  if (warp == NW) {
    // ===================================================== producer warp ==
    // Keeps every free ring slot loading; stores a batch as soon as its sweep 2
    // is done and refills the slot once the bulk engine has read it.
    if (lane != 0) return;
    const unsigned t_start = static_cast<unsigned>(globaltimer_ns());
    const uint64_t pol = a.evict_first ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_keep = policy_evict_last();
    // Iteration t = iter + 1 walks a static block backwards when t is odd: it
    // starts on the batches iteration t-1 (or the forward seed sweep) stored
    // last, still in L2 — their reads hit and their previous writes are
    // overwritten before reaching HBM.
    const bool snake = a.keep > 0 && !a.dyn && !SEED;
    const bool back = snake && ((ctl->iter + 1) & 1ull);
    BatchPick pick{ctl, a.mail + static_cast<size_t>(group) * kMail, r0, r1, (a.rows + B - 1) / B,
                   static_cast<unsigned long long>(ctl->sweep_seq) << 32, a.rows, B, G, g, nb_static,
                   // (the seed sweep has no row exchange to bound how far a leader runs
                   // ahead of its followers, so with G > 1 it keeps the static blocks)
                   a.dyn && !(SEED && G > 1), back};
    unsigned& nb = pick.nb;  // local batches with rows (known at the first sentinel)
    auto issue_load = [&](unsigned b) {
      const unsigned long long row = pick(b);
      uint64_t* bar = &full[b % NBUF];
      srow[b % NBUF] = row;
      if (row == kNoRow) {  // sentinel: the consumers stop here
        mbar_arrive(bar);
        return;
      }
      const unsigned nr = rows_at(row);
      T* dst = slot_ptr(b);
      const T* src = gbase + row_of(row) * a.pitch;
      mbar_arrive_expect_tx(bar, nr * row_bytes);
      if (G == 1) {
        bulk_g2s(dst, src, nr * row_bytes, bar, pol);  // rows contiguous when G == 1
      } else {
        for (unsigned r = 0; r < nr; ++r)
          bulk_g2s(dst + r * a.slice, src + static_cast<size_t>(r) * a.pitch, row_bytes, bar, pol);
      }
    };
    auto issue_store = [&](unsigned b) {
      const unsigned long long row = srow[b % NBUF];
      const unsigned nr = rows_at(row);
      const T* srcs = slot_ptr(b);
      T* dst = gbase + row_of(row) * a.pitch;
      const uint64_t sp = snake && b + a.keep >= nb_static ? pol_keep : pol;
      if (G == 1) {
        bulk_s2g(dst, srcs, nr * row_bytes, sp);
      } else {
        for (unsigned r = 0; r < nr; ++r)
          bulk_s2g(dst + static_cast<size_t>(r) * a.pitch, srcs + r * a.slice, row_bytes, sp);
      }
      bulk_commit();
    };
#ifdef UOT_TRACE
    const unsigned long long tr_p0 = clock64();
#endif
    // Sentinels go to local batches nb .. nb+NF-1: the compute warps stop at
    // nb, factor warp f at its first batch >= nb.
    for (unsigned b = 0; b < static_cast<unsigned>(NBUF); ++b) issue_load(b);
    for (unsigned b = 0; b < nb; ++b) {
      TR_BEGIN();
      mbar_wait(&done2[b % NBUF], (b / NBUF) & 1u);  // slot b consumed (sweep 2 / seed done)
      TR_END(4);
      if (SEED) {
        if (b + NBUF - NF < nb) issue_load(b + NBUF);
        continue;
      }
      issue_store(b);
      // refill the slot of the previous batch: its store has had a whole batch to drain
      if (b >= 1 && b - 1 + NBUF - NF < nb) {
        bulk_wait_read<1>();
        issue_load(b - 1 + NBUF);
      }
    }
    if (!SEED) bulk_wait<0>();  // every store landed before the CTA retires
    if (a.dbg) {
      a.dbg[kDbg * cta] = smid();
      a.dbg[kDbg * cta + 1] = nb;
      a.dbg[kDbg * cta + 2] = t_start;
      a.dbg[kDbg * cta + 3] = static_cast<unsigned>(globaltimer_ns());
    }
#ifdef UOT_TRACE
    atomicAdd(&uot_trace[8], clock64() - tr_p0);
    TR_FLUSH(4, 5);
#endif
    return;
  }

  if (warp > NW) {
    // ====================================================== factor warps ==
    // alpha_i = rescale_factor(rpd_i, s_i, fi) (fused.hpp:133) for every row,
    // ahead of the compute warps' sweep 2. NF warps take batches round robin so
    // the serial chain of one batch (partials, exchange round trip, pow) may
    // take NF batch-times.
    if (SEED) return;
    const unsigned f = static_cast<unsigned>(warp - NW - 1);
    const unsigned long long tag_hi = static_cast<unsigned long long>(ctl->epoch) << 32;
    double errmax = 0.0;
#ifdef UOT_TRACE
    const unsigned long long tr_f0 = clock64();
#endif
    for (unsigned s = f;; s += NF) {
      // the slot's first row (the slot cannot be refilled before this warp's alpha)
      mbar_wait(&full[s % NBUF], (s / NBUF) & 1u);
      const unsigned long long packed = srow[s % NBUF];
      if (packed == kNoRow) {
        // split roles: the sweep-2 warps learn the end from the factor ring (each
        // factor warp's first sentinel completes its slot's phase; only batch nb's is awaited)
        if (SPLIT && lane == 0) mbar_arrive(&alpha_rdy[s % QD]);
        break;
      }
      const unsigned nr = rows_at(packed);
      const unsigned long long row = row_of(packed);
      const unsigned q = s % QD;
      double rv = 0.0;
      if (lane < static_cast<int>(nr)) rv = __ldg(&a.rpd[row + lane]);
      TR_BEGIN();
      mbar_wait(&done1[q], (s / QD) & 1u);
      TR_END(0);
      double t = 0.0;  // this CTA's partial of row `lane` of the batch, warp order
      if (lane < static_cast<int>(nr)) {
        t = red[(q * NWR) * BM + lane];
#pragma unroll
        for (int w = 1; w < NWR; ++w) t += red[(q * NWR + w) * BM + lane];
      }
      if (XCHG) {
        TR_BEGIN();
        t = exchange_row_sum(a.xrec, cta, group, G, s % kRing, tag_hi | (s + 1), t, ctl);
        TR_END(2);
      }
      TR_BEGIN();
      double al = 0.0;
      if (lane < static_cast<int>(nr)) {
        if (!rescale_factor_dev(rv, t, a.fi, &al)) {
          atomicOr(&ctl->alpha_bad, 1);
          al = 1.0;
        }
        if (g == 0) {
          a.alpha[row + lane] = al;
          errmax = fmax(errmax, fabs(al - 1.0));
        }
      }
      // lane 0 — the thread that arrives on alpha_rdy — stores the batch's
      // factors itself (release by the arriving thread: no reliance on
      // __syncwarp cumulativity; compute-sanitizer racecheck clean)
#pragma unroll
      for (int r = 0; r < BM; ++r) {
        const double v = __shfl_sync(0xffffffffu, al, r);
        if (lane == 0 && r < static_cast<int>(nr)) alpha_s[q * BM + r] = v;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&alpha_rdy[q]);
      TR_END(3);
    }
    for (int o = 16; o > 0; o >>= 1) errmax = fmax(errmax, __shfl_xor_sync(0xffffffffu, errmax, o));
    if (lane == 0) {
      a.cta_err[kErrSlots * cta + f] = errmax;
      if (f == 0)
        for (int k = NF; k < kErrSlots; ++k) a.cta_err[kErrSlots * cta + k] = 0.0;
    }
#ifdef UOT_TRACE
    if (lane == 0 && f == 0) {
      TR_FLUSH(0, 4);
      atomicAdd(&uot_trace[9], clock64() - tr_f0);
    }
#endif
    return;
  }

  // ========================================================= compute warps ==
  if constexpr (SPLIT) {
    // Split roles. Threads [0, NT/2): sweep 1 of every batch over the whole
    // slice (chunks t + k*NT/2, k < 2V; factors in TMEM for V >= 3, else in
    // registers), the row partials and a per-row exact-path mask per warp.
    // Threads [NT/2, NT): sweep 2 of every batch once its factors are published,
    // and the column partials. Each warp waits on one barrier per batch and
    // keeps twice the independent work per wait.
    constexpr int NT2 = NT / 2, V2 = 2 * V, NW2 = NW / 2;
    const bool sweep1_role = tid < NT2;
    const unsigned t = sweep1_role ? tid : tid - NT2;
    const unsigned w = t >> 5;
    if (sweep1_role) {
      ScreenBounds sb1;
      const uint32_t tc = tbase + (static_cast<uint32_t>(32 * (w % 4)) << 16) + 8 * V2 * (w / 4);
      double beta[TB ? 1 : 4 * V2];  // (register factors: V2 <= 4)
      {
        double bl[4 * V2];
        const double* bsrc = a.beta2 + ((ctl->iter + 1) & 1ull) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
        for (int k = 0; k < V2; ++k) {
          const unsigned q = t + k * NT2;
#pragma unroll
          for (int e = 0; e < 4; ++e) bl[4 * k + e] = (FULL || q < nq) ? bsrc[4 * q + e] : 1.0;
        }
        sb1 = screen_bounds(bl, 4 * V2);
        if constexpr (TB) {
#pragma unroll
          for (int k = 0; k < V2; ++k) tmem_st_chunk(tc + 8 * k, bl + 4 * k);
          tmem_wait_st_();
        } else {
#pragma unroll
          for (int i = 0; i < 4 * V2; ++i) beta[i] = bl[i];
        }
      }
      for (unsigned s = 0;; ++s) {
        const unsigned slot = s % NBUF;
        mbar_wait(&full[slot], (s / NBUF) & 1u);
        if (srow[slot] == kNoRow) break;
        const unsigned nr = BM == 1 ? 1u : rows_at(srow[slot]);
        const unsigned q = s % QD;
        uint32_t badm = 0;
#pragma unroll
        for (int r = 0; r < BM; ++r) {
          if (r < static_cast<int>(nr)) {
            bool bad = false;
            float4* rowp = reinterpret_cast<float4*>(smem + slot * a.buf_stride) + r * (a.slice / 4);
            double part;
            if constexpr (TB)
              part = row_sweep1_tb<NT2, V2, FULL>(rowp, t, nq, tc, sb1, bad);
            else
              part = row_sweep1<NT2, V2, FULL>(rowp, t, nq, beta, sb1, bad);
            const double ts = warp_sum(part);
            if (__any_sync(0xffffffffu, bad)) badm |= 1u << r;
            if (lane == 0) red[(q * NW2 + w) * BM + r] = ts;
          }
        }
        if (lane == 0) xbad[q * NW2 + w] = badm;
        __syncwarp();
        if (lane == 0) mbar_arrive(&done1[q]);
      }
      if constexpr (TB) {
        tmem_fence_before_();
        asm volatile("bar.sync 1, %0;" ::"n"(NT2) : "memory");
        if (w == 0) {
          tmem_fence_after_();
          tmem_dealloc_cols<kTbCols>(tbase);
        }
      }
    } else {
      double acc2[4 * V2];
#pragma unroll
      for (int i = 0; i < 4 * V2; ++i) acc2[i] = 0.0;
      for (unsigned b = 0;; ++b) {
        const unsigned q = b % QD, slot = b % NBUF;
        mbar_wait(&alpha_rdy[q], (b / QD) & 1u);
        if (srow[slot] == kNoRow) break;  // (the factor warps' sentinel completed this phase)
        const unsigned nr = BM == 1 ? 1u : rows_at(srow[slot]);
        const uint32_t badm = xbad[q * NW2 + w];
#pragma unroll
        for (int r = 0; r < BM; ++r)
          if (r < static_cast<int>(nr))
            row_sweep2<NT2, V2, FULL>(reinterpret_cast<float4*>(smem + slot * a.buf_stride) + r * (a.slice / 4), t,
                                      nq, alpha_s[q * BM + r], (badm >> r) & 1u, acc2);
        fence_proxy_async_smem();  // generic writes -> the producer's bulk store
        __syncwarp();
        if (lane == 0) mbar_arrive(&done2[slot]);
      }
      double* dst = a.partials + static_cast<size_t>(group) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
      for (int k = 0; k < V2; ++k) {
        const unsigned q = t + k * NT2;
        if (q < nq) {
          reinterpret_cast<double2*>(dst)[2 * q] = make_double2(acc2[4 * k], acc2[4 * k + 1]);
          reinterpret_cast<double2*>(dst)[2 * q + 1] = make_double2(acc2[4 * k + 2], acc2[4 * k + 3]);
        }
      }
    }
    return;
  } else {
  double beta[EPC * V], acc[EPC * V];
#pragma unroll
  for (int i = 0; i < EPC * V; ++i) acc[i] = 0.0;
  ScreenBounds sb{0xffffffffu, 0u};
  if (!SEED) {
    const double* bsrc = a.beta2 + ((ctl->iter + 1) & 1ull) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = tid + k * NT;
#pragma unroll
      for (int e = 0; e < EPC; ++e) beta[EPC * k + e] = (FULL || q < nq) ? bsrc[EPC * q + e] : 1.0;
    }
    if (!F64) sb = screen_bounds(beta, EPC * V);
  }
  // this thread's TMEM factor columns (TB): lane quarter warp%4, column block warp/4
  const uint32_t tcol = tbase + (static_cast<uint32_t>(32 * (warp % 4)) << 16) + 8 * V * (warp / 4);
  if (TB) {
#pragma unroll
    for (int k = 0; k < V; ++k) tmem_st_chunk(tcol + 8 * k, beta + 4 * k);
    tmem_wait_st_();
  }

#ifdef UOT_TRACE
  const unsigned long long tr_c0 = clock64();
#endif
  if (SEED) {
    for (unsigned s = 0;; ++s) {
      mbar_wait(&full[s % NBUF], (s / NBUF) & 1u);
      if (srow[s % NBUF] == kNoRow) break;
      const T* buf = slot_ptr(s);
      const unsigned nr = rows_at(srow[s % NBUF]);
#pragma unroll
      for (int r = 0; r < BM; ++r)
        if (r < static_cast<int>(nr)) {
          if constexpr (F64)
            row_seed_f64<NT, V, FULL>(reinterpret_cast<const double2*>(buf + r * a.slice), tid, nq, acc);
          else
            row_seed<NT, V, FULL>(reinterpret_cast<const float4*>(buf + r * a.slice), tid, nq, acc);
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&done2[s % NBUF]);
    }
  } else {
    // bit (b % 8) * BM + r: row r of batch b took the exact path in sweep 1
    using Mask = typename std::conditional<(BM <= 4), uint32_t, uint64_t>::type;
    Mask x1bad = 0;
    unsigned nb = 0xffffffffu;        // local batches (set at the sentinel)
    unsigned slot1 = 0, ph1 = 0;      // ring slot and full-barrier parity of batch s
    unsigned slot2 = 0;               // ring slot of batch b = s - LA - 1
    for (unsigned s = 0;; ++s) {
      bool s1 = s < nb;  // sweep 1 of batch s
      if (s1) {
        TR_BEGIN();
        mbar_wait(&full[slot1], ph1);
        TR_END(16);
        if (srow[slot1] == kNoRow) {
          nb = s;
          s1 = false;
        }
      }
      const bool s2 = s >= static_cast<unsigned>(LA + 1) && s - (LA + 1) < nb;  // sweep 2 of batch b
      if (!s1 && s >= nb + LA + 1) break;  // (nb is known once s1 is false)
      const unsigned b = s - (LA + 1);
      double part[BM];
      if (s1) {
        T* buf = reinterpret_cast<T*>(smem + slot1 * a.buf_stride);
        const unsigned nr = BM == 1 ? 1u : rows_at(srow[slot1]);
        const unsigned sh = (s % 8) * BM;
        x1bad &= ~(static_cast<Mask>((1u << BM) - 1u) << sh);
#pragma unroll
        for (int r = 0; r < BM; ++r) {
          part[r] = 0.0;
          if (r < static_cast<int>(nr)) {
            if constexpr (F64) {
              part[r] = row_sweep1_f64<NT, V, FULL>(reinterpret_cast<double2*>(buf + r * a.slice), tid, nq, beta);
            } else {
              bool bad = false;
              if constexpr (TB)
                part[r] = row_sweep1_tb<NT, V, FULL>(reinterpret_cast<float4*>(buf + r * a.slice), tid, nq, tcol,
                                                     sb, bad);
              else
                part[r] =
                    row_sweep1<NT, V, FULL>(reinterpret_cast<float4*>(buf + r * a.slice), tid, nq, beta, sb, bad);
              if (bad) x1bad |= static_cast<Mask>(1u) << (sh + r);
            }
          }
        }
      }
      if (s2) {  // sweep 2 of batch s-1-LA once its factors are published
        TR_BEGIN();
        mbar_wait(&alpha_rdy[b % kQ], (b / kQ) & 1u);  // (plain / nanosleep polls: measured no faster)
        TR_END(19);
        T* buf = reinterpret_cast<T*>(smem + slot2 * a.buf_stride);
        const unsigned nr = BM == 1 ? 1u : rows_at(srow[slot2]);
        const unsigned sh = (b % 8) * BM;
#pragma unroll
        for (int r = 0; r < BM; ++r)
          if (r < static_cast<int>(nr)) {
            if constexpr (F64)
              row_sweep2_f64<NT, V, FULL>(reinterpret_cast<double2*>(buf + r * a.slice), tid, nq,
                                          alpha_s[(b % kQ) * BM + r], acc);
            else
              row_sweep2<NT, V, FULL>(reinterpret_cast<float4*>(buf + r * a.slice), tid, nq,
                                      alpha_s[(b % kQ) * BM + r], (x1bad >> (sh + r)) & 1u, acc);
          }
        fence_proxy_async_smem();  // generic writes -> the producer's bulk store
        __syncwarp();
        if (lane == 0) mbar_arrive(&done2[slot2]);
        slot2 = slot2 + 1 == NBUF ? 0 : slot2 + 1;
      }
      if (s1) {  // row partials of batch s (after sweep 2, whose work hides the shuffle latency)
        const unsigned qq = s % kQ;
        const unsigned nr = BM == 1 ? 1u : rows_at(srow[slot1]);
#pragma unroll
        for (int r = 0; r < BM; ++r) {
          if (r < static_cast<int>(nr)) {
            const double t = warp_sum(part[r]);
            if (lane == 0) red[(qq * NW + warp) * BM + r] = t;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&done1[qq]);
      }
      if (++slot1 == NBUF) {
        slot1 = 0;
        ph1 ^= 1u;
      }
    }
  }
  if (TB) {  // every compute warp is done with TMEM: compute warp 0 frees it
    tmem_fence_before_();
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    if (warp == 0) {
      tmem_fence_after_();
      tmem_dealloc_cols<kTbCols>(tbase);
    }
  }
#ifdef UOT_TRACE
  if (tid == 0) {
    TR_FLUSH(16, 20);
    atomicAdd(&uot_trace[21], clock64() - tr_c0);
  }
#endif

  // Column partials of this CTA: one row of the [groups][pitch] table.
  double* dst = a.partials + static_cast<size_t>(group) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const unsigned q = tid + k * NT;
    if (q < nq) {
#pragma unroll
      for (int h = 0; h < EPC / 2; ++h)
        reinterpret_cast<double2*>(dst)[(EPC / 2) * q + h] =
            make_double2(acc[EPC * k + 2 * h], acc[EPC * k + 2 * h + 1]);
    }
  }
  }  // !SPLIT
}

}  // namespace uotk
