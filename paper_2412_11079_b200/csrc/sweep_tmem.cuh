// sweep_tmem.cuh — the fused MAP-UOT iteration with the alpha-lag parked in TMEM.
//
// Same arithmetic and reference lines as sweep.cuh (fused_row_pass,
// fused.hpp:119-144); what changes is where a row waits for its factor.
// Between sweep 1 (x1 = f32(x0*beta), row partial) and sweep 2 (x2 =
// f32(x1*alpha)) a row must be held until alpha_i is known — with G > 1 CTAs per
// row that includes a cross-CTA exchange through L2 whose latency varies with
// the skew between the CTAs of a group. In sweep.cuh the waiting rows occupy the
// shared-memory ring (7 x 32 KiB), which caps the lag at 2 batches. Here the
// waiting x1 values are parked in Tensor Memory (256 KB per SM, otherwise unused
// by this bandwidth-bound kernel): each compute thread writes its 4*V*BM values
// of a batch to its own TMEM lane with tcgen05.st and reads them back for sweep 2
// with tcgen05.ld. Shared memory then only holds a LOAD ring (TMA in, sweep 1
// reads) and a STORE ring (sweep 2 writes, bulk copy out), and the lag between
// the sweeps can be up to TQ - 2 batches (TQ = TMEM slots, 8 for 64 columns per
// batch) without costing a byte of shared memory.
//
// Roles (one CTA per SM, persistent over its row block):
//   producer warp  TMEM alloc/dealloc; lane 0 streams batches into the load ring
//                  (cp.async.bulk, mbarrier complete_tx) as soon as sweep 1 has
//                  read a slot, and bulk-stores finished batches from the store
//                  ring, in the compute warps' step order.
//   compute warps  step s: sweep 1 of batch s (smem -> regs -> TMEM), row
//                  partials -> done1(s); sweep 2 of batch s-LA-1 (TMEM -> regs ->
//                  store ring), column partials in registers.
//   factor warps   alpha_i = rescale_factor(rpd_i, s_i, fi) per row, after the
//                  cross-CTA exchange of row partials when G > 1 (as sweep.cuh).
#pragma once
#include <cstdint>

#include "sweep.cuh"

namespace uotk {

constexpr int kQT = 8;          // done1 / alpha ring depth (>= LA + 2)
constexpr int kTmemCols = 512;  // the whole TMEM of the SM (one CTA per SM)

// ------------------------------------------------------------- tcgen05 --
__device__ __forceinline__ void tmem_alloc_512(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst_smem))
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_512(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 bit, 4 consecutive columns per thread (one float4).
__device__ __forceinline__ void tmem_st4(uint32_t taddr, float4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
               "r"(__float_as_uint(v.w))
               : "memory");
}
__device__ __forceinline__ float4 tmem_ld4(uint32_t taddr) {
  uint32_t x, y, z, w;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
               : "r"(taddr)
               : "memory");
  return make_float4(__uint_as_float(x), __uint_as_float(y), __uint_as_float(z), __uint_as_float(w));
}

// ---------------------------------------------------- per-row bodies --
// The arithmetic of sweep.cuh's bodies (window screen certifying x0 and x1,
// two-op widening, hardware widening for the column sums); only where x1 waits
// differs: TMEM columns [tcol, tcol + 4V) of this thread's lane.

// fused.hpp:125-131: x1 = f32(f64(x0)*beta_j) from the load slot into TMEM;
// returns the f64 row partial; `bad` when a group took the exact path.
template <int NT, int V, bool FULL>
__device__ __forceinline__ double row_sweep1_t(const float4* row, uint32_t tcol, unsigned tid, unsigned nq,
                                               const double* beta, ScreenBounds sb, bool& bad) {
  constexpr int KG = ChunkGroup<V>::KG;
  double s[4];
#pragma unroll
  for (int g0 = 0; g0 < V; g0 += KG) {
    float4 v[KG];
    load_group<NT, KG, FULL>(row, v, g0, tid, nq);
    const uint32_t m = screen_group<KG>(v, sb.lo);
    double t[4];
    if (m <= sb.span) {
#pragma unroll
      for (int kk = 0; kk < KG; ++kk)
#pragma unroll
        for (int e = 0; e < 4; ++e) comp(v[kk], e) = d2f(fastd(comp(v[kk], e)) * beta[4 * (g0 + kk) + e]);
#pragma unroll
      for (int e = 0; e < 4; ++e) t[e] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KG; ++kk)
        if (FULL || tid + (g0 + kk) * NT < nq)
#pragma unroll
          for (int e = 0; e < 4; ++e) t[e] += fastd(comp(v[kk], e));
    } else {
      bad = true;
#pragma unroll
      for (int kk = 0; kk < KG; ++kk)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          comp(v[kk], e) = d2f(static_cast<double>(comp(v[kk], e)) * beta[4 * (g0 + kk) + e]);
#pragma unroll
      for (int e = 0; e < 4; ++e) t[e] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KG; ++kk)
        if (FULL || tid + (g0 + kk) * NT < nq)
#pragma unroll
          for (int e = 0; e < 4; ++e) t[e] += static_cast<double>(comp(v[kk], e));
    }
    __syncwarp();  // tcgen05.st is warp-collective (.sync.aligned)
#pragma unroll
    for (int kk = 0; kk < KG; ++kk) tmem_st4(tcol + 4 * (g0 + kk), v[kk]);
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = g0 == 0 ? t[e] : s[e] + t[e];
  }
  return (s[0] + s[1]) + (s[2] + s[3]);
}

// fused.hpp:135-142: x2 = f32(f64(x1)*alpha) from TMEM into the store slot,
// next_j += f64(x2).
template <int NT, int V, bool FULL>
__device__ __forceinline__ void row_sweep2_t(uint32_t tcol, float4* out, unsigned tid, unsigned nq, double al,
                                             bool exact, double* acc) {
  constexpr int KG = ChunkGroup<V>::KG;
  float4 v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) v[k] = tmem_ld4(tcol + 4 * k);
  tmem_wait_ld();
#pragma unroll
  for (int g0 = 0; g0 < V; g0 += KG) {
    float4 (&w)[KG] = *reinterpret_cast<float4(*)[KG]>(&v[g0]);
    if (exact)
      group_sweep2<NT, KG, FULL, true>(out, w, g0, tid, nq, al, acc);
    else
      group_sweep2<NT, KG, FULL, false>(out, w, g0, tid, nq, al, acc);
  }
}

// Shared-memory layout shared by host sizing and the kernel.
template <int NW, int BM, int NL, int NS>
struct TmemSweepSmem {
  static constexpr int kBars = 2 * NL + 2 * NS + 2 * kQT;
  static constexpr int kDoubles = kQT * NW * BM /*red*/ + kQT * BM /*alpha*/;
  static size_t bytes(unsigned buf_stride) {
    return static_cast<size_t>(NL + NS) * buf_stride + kBars * 8 + 16 /*tmem base*/ + kDoubles * 8;
  }
};

template <int NT, int V, int BM>
struct TmemGeometry {
  static constexpr int NW = NT / 32;
  static constexpr int kColsPerWarp = 4 * V * BM;             // one batch of one thread
  static constexpr int kColsPerSlot = (NW / 4) * kColsPerWarp;  // 4 warps share a lane quarter
  static constexpr int TQ = kTmemCols / kColsPerSlot > 32 ? 32 : kTmemCols / kColsPerSlot;
  static_assert(NW % 4 == 0, "compute warps must cover the four TMEM lane quarters evenly");
};

// NT compute threads + producer warp + NF factor warps; NL load / NS store ring
// slots; LA extra batches between sweep 1 and sweep 2 (kept in TMEM).
// S2FIRST: a step runs sweep 2 of the oldest batch before sweep 1 of the newest,
// so tcgen05.wait::st only waits for TMEM stores issued a whole sweep earlier.
template <int NT, int V, int BM, int NL, int NS, int LA, bool XCHG, int NF, bool FULL, bool S2FIRST = true>
__global__ void __launch_bounds__(NT + 32 * (1 + NF), 1) sweep_tmem_kernel(const SweepArgs a) {
  using Geo = TmemGeometry<NT, V, BM>;
  constexpr int NW = NT / 32;
  static_assert(NF >= 1 && NF <= kErrSlots, "factor warps");
  static_assert(LA >= 1 && LA + 2 <= Geo::TQ && LA + 2 <= kQT, "lag exceeds the TMEM / factor rings");
  static_assert(NL >= 2 && NS >= 2, "rings");
  static_assert(!XCHG || BM == 1, "the exchange path moves one row per batch");

  extern __shared__ __align__(128) unsigned char smem[];
  Control* ctl = a.ctl;
  if (ctl->done) return;
  if (ctl->beta_bad) {  // beta_from_state threw at the top of this iteration
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(&ctl->status, kStatusDegenerateBeta);
      ctl->done = 1;
    }
    return;
  }

  unsigned char* const lring = smem;
  unsigned char* const sring = smem + NL * a.buf_stride;
  uint64_t* lfull = reinterpret_cast<uint64_t*>(smem + (NL + NS) * a.buf_stride);
  uint64_t* lfree = lfull + NL;
  uint64_t* sfull = lfree + NL;
  uint64_t* sfree = sfull + NS;
  uint64_t* done1 = sfree + NS;
  uint64_t* alpha_rdy = done1 + kQT;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(alpha_rdy + kQT);
  double* red = reinterpret_cast<double*>(tmem_base_s + 4);  // [kQT][NW][BM]
  double* alpha_s = red + kQT * NW * BM;                     // [kQT][BM]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned G = a.G;
  const unsigned cta = a.smid_map ? smid() : blockIdx.x;
  const unsigned group = cta / G, g = cta % G;
  const unsigned long long base = a.rows / a.groups, rem = a.rows % a.groups;  // plan.cpp:11-21
  const unsigned long long r0 = group * base + (group < rem ? group : rem);
  const unsigned nrows = static_cast<unsigned>(base + (group < rem ? 1 : 0));
  const unsigned B = a.B;
  const unsigned nb = (nrows + B - 1) / B;
  const unsigned nq = a.slice >> 2;
  const uint32_t row_bytes = a.slice * 4u;
  float* gbase = static_cast<float*>(a.P) + r0 * a.pitch + static_cast<size_t>(g) * a.slice;
  auto rows_in = [&](unsigned b) -> unsigned { return min(B, nrows - b * B); };
  auto lslot = [&](unsigned b) -> float* { return reinterpret_cast<float*>(lring + (b % NL) * a.buf_stride); };
  auto sslot = [&](unsigned b) -> float* { return reinterpret_cast<float*>(sring + (b % NS) * a.buf_stride); };

  if (tid == 0) {
    for (int i = 0; i < NL; ++i) {
      mbar_init(&lfull[i], 1);
      mbar_init(&lfree[i], NW);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&sfull[i], NW);
      mbar_init(&sfree[i], 1);
    }
    for (int i = 0; i < kQT; ++i) {
      mbar_init(&done1[i], NW);
      mbar_init(&alpha_rdy[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == NW) tmem_alloc_512(tmem_base_s);  // whole producer warp (warp-collective)
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tmem_base_s;

  if (warp == NW) {
    // ===================================================== producer warp ==
    if (lane == 0) {
      const uint64_t pol = a.evict_first ? policy_evict_first() : policy_evict_normal();
      auto issue_load = [&](unsigned b) {
        const unsigned nr = rows_in(b);
        uint64_t* bar = &lfull[b % NL];
        float* dst = lslot(b);
        const float* src = gbase + static_cast<size_t>(b) * B * a.pitch;
        mbar_arrive_expect_tx(bar, nr * row_bytes);
        if (G == 1) {
          bulk_g2s(dst, src, nr * row_bytes, bar, pol);  // rows contiguous when G == 1
        } else {
          for (unsigned r = 0; r < nr; ++r)
            bulk_g2s(dst + r * a.slice, src + static_cast<size_t>(r) * a.pitch, row_bytes, bar, pol);
        }
      };
      for (unsigned b = 0; b < nb && b < static_cast<unsigned>(NL); ++b) issue_load(b);
      // Follow the compute warps' step order: sweep 1 of s frees load slot s,
      // sweep 2 of s-LA-1 fills a store slot.
      auto refill = [&](unsigned s) {  // sweep 1 of s has read its load slot
        mbar_wait(&lfree[s % NL], (s / NL) & 1u);
        if (s + NL < nb) issue_load(s + NL);
      };
      auto store = [&](unsigned b) {  // sweep 2 of b has filled its store slot
        mbar_wait(&sfull[b % NS], (b / NS) & 1u);
        const unsigned nr = rows_in(b);
        const float* srcs = sslot(b);
        float* dst = gbase + static_cast<size_t>(b) * B * a.pitch;
        if (G == 1) {
          bulk_s2g(dst, srcs, nr * row_bytes, pol);
        } else {
          for (unsigned r = 0; r < nr; ++r)
            bulk_s2g(dst + static_cast<size_t>(r) * a.pitch, srcs + r * a.slice, row_bytes, pol);
        }
        bulk_commit();
        if (b >= 1) {  // the previous store has been read out of its slot: hand it back
          bulk_wait_read<1>();
          mbar_arrive(&sfree[(b - 1) % NS]);
        }
      };
      // Follow the compute warps' step order exactly (no deadlock by construction).
      for (unsigned s = 0; s < nb + LA + 1; ++s) {
        const bool s2 = s >= static_cast<unsigned>(LA + 1) && s - (LA + 1) < nb;
        if (S2FIRST && s2) store(s - (LA + 1));
        if (s < nb) refill(s);
        if (!S2FIRST && s2) store(s - (LA + 1));
      }
      bulk_wait<0>();  // every store landed before the CTA retires
    }
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"n"(NT + 32) : "memory");  // compute warps are done with TMEM
    tmem_fence_after();
    tmem_dealloc_512(tbase);
    return;
  }

  if (warp > NW) {
    // ====================================================== factor warps ==
    // alpha_i = rescale_factor(rpd_i, s_i, fi) (fused.hpp:133) for every row of
    // a batch; NF warps take batches round robin (see sweep.cuh).
    const unsigned f = static_cast<unsigned>(warp - NW - 1);
    const unsigned long long tag_hi = static_cast<unsigned long long>(ctl->epoch) << 32;
    double errmax = 0.0;
    for (unsigned s = f; s < nb; s += NF) {
      const unsigned nr = rows_in(s);
      const unsigned q = s % kQT;
      double rv = 0.0;
      if (lane < static_cast<int>(nr)) rv = __ldg(&a.rpd[r0 + static_cast<unsigned long long>(s) * B + lane]);
      mbar_wait(&done1[q], (s / kQT) & 1u);
      double t = 0.0;  // this CTA's partial of row `lane` of the batch, warp order
      if (lane < static_cast<int>(nr)) {
        t = red[(q * NW) * BM + lane];
#pragma unroll
        for (int w = 1; w < NW; ++w) t += red[(q * NW + w) * BM + lane];
      }
      if (XCHG) t = exchange_row_sum(a.xrec, cta, group, G, s % kRing, tag_hi | (s + 1), t, ctl);

      double al = 0.0;
      if (lane < static_cast<int>(nr)) {
        if (!rescale_factor_dev(rv, t, a.fi, &al)) {
          atomicOr(&ctl->alpha_bad, 1);
          al = 1.0;
        }
        if (g == 0) {
          a.alpha[r0 + static_cast<unsigned long long>(s) * B + lane] = al;
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
    }
    for (int o = 16; o > 0; o >>= 1) errmax = fmax(errmax, __shfl_xor_sync(0xffffffffu, errmax, o));
    if (lane == 0) {
      a.cta_err[kErrSlots * cta + f] = errmax;
      if (f == 0)
        for (int k = NF; k < kErrSlots; ++k) a.cta_err[kErrSlots * cta + k] = 0.0;
    }
    return;
  }

  // ========================================================= compute warps ==
  double beta[4 * V], acc[4 * V];
#pragma unroll
  for (int i = 0; i < 4 * V; ++i) acc[i] = 0.0;
  {
    const double* bsrc = a.beta2 + ((ctl->iter + 1) & 1ull) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = tid + k * NT;
#pragma unroll
      for (int e = 0; e < 4; ++e) beta[4 * k + e] = (FULL || q < nq) ? bsrc[4 * q + e] : 1.0;
    }
  }
  const ScreenBounds sb = screen_bounds(beta, 4 * V);
  // TMEM address of (batch slot, row r) for this thread: lane quarter warp%4,
  // column block (warp/4) within the slot.
  const uint32_t tlane = static_cast<uint32_t>(32 * (warp & 3)) << 16;
  auto tcol = [&](unsigned b, int r) -> uint32_t {
    return tbase + tlane + (b % Geo::TQ) * Geo::kColsPerSlot + (warp >> 2) * Geo::kColsPerWarp + r * 4 * V;
  };

  uint64_t x1bad = 0;  // bit (b % 8) * 8 + r: row r of batch b stored a non-normal x1
  // sweep 1 of batch s: load slot -> TMEM, row partials -> done1(s)
  auto sweep1 = [&](unsigned s) {
      mbar_wait(&lfull[s % NL], (s / NL) & 1u);
      const float* buf = lslot(s);
      const unsigned nr = rows_in(s);
      const uint32_t shift = (s % 8) * 8;
      x1bad &= ~(0xffull << shift);
      double part[BM];
#pragma unroll
      for (int r = 0; r < BM; ++r) {
        part[r] = 0.0;
        if (r < static_cast<int>(nr)) {
          bool bad = false;
          part[r] = row_sweep1_t<NT, V, FULL>(reinterpret_cast<const float4*>(buf + r * a.slice), tcol(s, r), tid,
                                              nq, beta, sb, bad);
          if (bad) x1bad |= 1ull << (shift + r);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&lfree[s % NL]);  // slot read: the producer may refill it
      const unsigned qq = s % kQT;
#pragma unroll
      for (int r = 0; r < BM; ++r) {
        if (r < static_cast<int>(nr)) {
          const double t = warp_sum(part[r]);
          if (lane == 0) red[(qq * NW + warp) * BM + r] = t;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&done1[qq]);
  };
  // sweep 2 of batch b = s-LA-1: TMEM -> store slot, column partials
  auto sweep2 = [&](unsigned s) {
      const unsigned b = s - (LA + 1);
      const unsigned qb = b % kQT;
      mbar_wait(&alpha_rdy[qb], (b / kQT) & 1u);
      if (b >= static_cast<unsigned>(NS)) mbar_wait(&sfree[b % NS], ((b / NS) - 1) & 1u);
      tmem_wait_st();  // this thread's x1 of batch b is in TMEM
      float* out = sslot(b);
      const unsigned nr = rows_in(b);
      const uint32_t shift = (b % 8) * 8;
#pragma unroll
      for (int r = 0; r < BM; ++r)
        if (r < static_cast<int>(nr))
          row_sweep2_t<NT, V, FULL>(tcol(b, r), reinterpret_cast<float4*>(out + r * a.slice), tid, nq,
                                    alpha_s[qb * BM + r], (x1bad >> (shift + r)) & 1ull, acc);
      fence_proxy_async_smem();  // generic writes -> the producer's bulk store
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[b % NS]);
  };
  for (unsigned s = 0; s < nb + LA + 1; ++s) {
    const bool s2 = s >= static_cast<unsigned>(LA + 1) && s - (LA + 1) < nb;
    if (S2FIRST && s2) sweep2(s);
    if (s < nb) sweep1(s);
    if (!S2FIRST && s2) sweep2(s);
  }
  tmem_fence_before();
  asm volatile("bar.sync 1, %0;" ::"n"(NT + 32) : "memory");

  // Column partials of this CTA: one row of the [groups][pitch] table.
  double* dst = a.partials + static_cast<size_t>(group) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const unsigned q = tid + k * NT;
    if (q < nq) {
      reinterpret_cast<double2*>(dst)[2 * q] = make_double2(acc[4 * k + 0], acc[4 * k + 1]);
      reinterpret_cast<double2*>(dst)[2 * q + 1] = make_double2(acc[4 * k + 2], acc[4 * k + 3]);
    }
  }
}

}  // namespace uotk
