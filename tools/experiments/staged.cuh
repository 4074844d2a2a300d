// staged.cuh — the fused iteration with the alpha lag held in Tensor Memory.
// EXPERIMENT (not built into the product): measured on B200 with
// 5 load + 2 store slots, 6 TMEM row slots: 32768^2 +-0..+1%, 8192^2 +2% slower
// than the split-role ring kernel; 4 + 3 slots +2..3% slower. To try it, include
// it after sweep.cuh in uot_cuda.cu and point make_cfg's iter[] of the V >= 3,
// BM == 1 configurations at staged_kernel<NT, V, NL, NB - NL, XCHG, NF, FULL>
// (dynamic smem = max(SweepSmem, StagedSmem)).
//
// Same arithmetic, order of additions and outputs as sweep_kernel's split-role
// path (sweep.cuh; fused.hpp:119-144 per row, 242-248 for the partials); what
// changes is where a row waits for its factor alpha_i:
//
//   load slot (smem) --sweep 1--> TMEM row slot --alpha--> sweep 2 --> store slot (smem) --> HBM
//
//   * sweep-1 warps read x0 from a LOAD slot, write x1 = f32(f64(x0)*beta_j)
//     into their TMEM lanes (tcgen05.st) and free the load slot at once, so the
//     producer keeps NL - 1 loads in flight whatever the factor latency (the
//     G-CTA row-sum exchange through L2 for G > 1);
//   * sweep-2 warps (same TMEM lane quarter and columns as their sweep-1
//     partner warp) read x1 back (tcgen05.ld) once alpha_i is published, write
//     x2 into a STORE slot and free the TMEM row slot;
//   * the producer thread issues loads into free load slots and bulk stores
//     from filled store slots, polling both rings.
//
// TMEM per lane quarter (512 columns): the sweep-1 factors beta_j (2 warps x
// 8*V2 columns), then NTM row slots of 2 warps x 4*V2 columns of x1.
#pragma once
#include "../../paper_2412_11079_b200/csrc/sweep.cuh"

namespace uotk {

#ifndef UOT_STAGED_H
#define UOT_STAGED_H 4
#endif
constexpr int kStQ = 12;     // done1 / alpha rings: > NTM + NF, a multiple of NF (2, 3)
constexpr int kStRows = 16;  // the producer's batch-row ring: > batches between a load and its store

template <int V>
struct StagedTmem {
  static constexpr int V2 = 2 * V;             // float4 chunks per thread and role
  static constexpr int kFactorCols = 16 * V2;  // per quarter: 2 warps x V2 chunks x 8 columns (4 doubles)
  static constexpr int kRowCols = 8 * V2;      // per quarter: 2 warps x V2 chunks x 4 columns (4 floats)
  static constexpr int NTM = (512 - kFactorCols) / kRowCols > 8 ? 8 : (512 - kFactorCols) / kRowCols;
  static_assert(NTM >= 3, "TMEM row slots");
};

template <int NL, int NS>
struct StagedSmem {
  static constexpr int kBars = NL /*full*/ + NL /*lfree*/ + NS /*sfull*/ + NS /*sfree*/ + 8 /*tfree*/ +
                               kStQ /*done1*/ + kStQ /*alpha_rdy*/;
  static constexpr int kWords = kStQ * 8 /*red*/ + kStQ /*alpha*/ + kStRows /*rows*/ + kStQ * 4 /*xbad*/ + 1;
  static size_t bytes(unsigned buf_stride) {
    return static_cast<size_t>(NL + NS) * buf_stride + kBars * 8 + kWords * 8;
  }
};

__device__ __forceinline__ void tmem_st_x8f(uint32_t taddr, const float4& a, const float4& b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
               : "memory");
}
__device__ __forceinline__ void tmem_ld_x8f(uint32_t taddr, float4& a, float4& b) {  // (no wait)
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "r"(taddr)
               : "memory");
}

// NT compute threads (NT/2 per role), V float4 chunks per thread of the
// one-role-per-warp layout (each role covers 2V), NL load + NS store slots of
// one row slice, NF factor warps; fp32 storage, factors in TMEM.
template <int NT, int V, int NL, int NS, bool XCHG, int NF, bool FULL>
__global__ void __launch_bounds__(NT + 32 * (1 + NF), 1) staged_kernel(const SweepArgs a) {
  constexpr int NW = NT / 32, NT2 = NT / 2, NW2 = NW / 2, V2 = 2 * V;
  constexpr int NTM = StagedTmem<V>::NTM, FCOLS = StagedTmem<V>::kFactorCols, RCOLS = StagedTmem<V>::kRowCols;
  constexpr int KG = 2;  // chunks per group: one tcgen05 .x8 of x1 per group
  static_assert(NW2 == 8 && V2 % KG == 0 && kStQ % NF == 0 && kStQ > NTM + NF, "staged layout");
  static_assert(NL >= 3 && NS >= 2, "rings");

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
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (NL + NS) * a.buf_stride);
  uint64_t* lfree = full + NL;
  uint64_t* sfull = lfree + NL;
  uint64_t* sfree = sfull + NS;
  uint64_t* tfree = sfree + NS;
  uint64_t* done1 = tfree + 8;
  uint64_t* alpha_rdy = done1 + kStQ;
  double* red = reinterpret_cast<double*>(alpha_rdy + kStQ);  // [kStQ][NW2]
  double* alpha_s = red + kStQ * NW2;                          // [kStQ]  (< 0: no batch left)
  unsigned long long* rowq = reinterpret_cast<unsigned long long*>(alpha_s + kStQ);  // [kStRows]
  uint32_t* xbad = reinterpret_cast<uint32_t*>(rowq + kStRows);                     // [kStQ][NW2]
  uint32_t* tmem_s = xbad + kStQ * NW2;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned G = a.G;
  const unsigned cta = a.slot_of_sm ? a.slot_of_sm[smid()] : (a.smid_map ? smid() : blockIdx.x);
  const unsigned group = cta / G, g = cta % G;
  const unsigned B = a.B;  // 1: one row slice per batch
  const unsigned long long base = a.rows / a.groups, rem = a.rows % a.groups;
  const unsigned long long r0 = a.gbounds ? a.gbounds[group] : group * base + (group < rem ? group : rem);
  const unsigned long long r1 = a.gbounds ? a.gbounds[group + 1] : r0 + base + (group < rem ? 1 : 0);
  const unsigned nb_static = static_cast<unsigned>((r1 - r0 + B - 1) / B);
  const unsigned nq = a.slice / 4;
  const uint32_t row_bytes = a.slice * 4u;
  float* gbase = static_cast<float*>(a.P) + static_cast<size_t>(g) * a.slice;

  if (tid == 0) {
    for (int i = 0; i < NL; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&lfree[i], NW2);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&sfull[i], NW2);
      mbar_init(&sfree[i], 1);
    }
    for (int i = 0; i < NTM; ++i) mbar_init(&tfree[i], NW2);
    for (int i = 0; i < kStQ; ++i) {
      mbar_init(&done1[i], NW2);
      mbar_init(&alpha_rdy[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_cols<512>(tmem_s);
  tmem_fence_before_();
  __syncthreads();
  tmem_fence_after_();
  const uint32_t tbase = *tmem_s;

  if (warp == NW) {
    // ===================================================== producer thread ==
    if (lane != 0) return;
    const unsigned t_start = static_cast<unsigned>(globaltimer_ns());
    const uint64_t pol = a.evict_first ? policy_evict_first() : policy_evict_normal();
    const uint64_t pol_keep = policy_evict_last();
    const bool snake = a.keep > 0 && !a.dyn;
    const bool back = snake && ((ctl->iter + 1) & 1ull);
    BatchPick pick{ctl, a.mail + static_cast<size_t>(group) * kMail, r0, r1, (a.rows + B - 1) / B,
                   static_cast<unsigned long long>(ctl->sweep_seq) << 32, a.rows, B, G, g, nb_static,
                   a.dyn != 0, back};
    unsigned nl = 0, ns = 0;
    bool loads_done = false;
    auto issue_load = [&](unsigned b) {
      const unsigned long long row = pick(b);
      uint64_t* bar = &full[b % NL];
      if (row == kNoRow) {  // sentinel: sweep-1 warps stop here, factor warps at b .. b+NF-1
        for (int i = 0; i < NF; ++i) rowq[(b + i) % kStRows] = kNoRow;
        mbar_arrive(bar);
        loads_done = true;
        return;
      }
      rowq[b % kStRows] = row;
      mbar_arrive_expect_tx(bar, row_bytes);
      bulk_g2s(smem + (b % NL) * a.buf_stride, gbase + row_of_batch(row) * a.pitch, row_bytes, bar, pol);
    };
    while (nl < static_cast<unsigned>(NL) && !loads_done) issue_load(nl++);
    for (;;) {
      if (!loads_done && mbar_try_wait(&lfree[nl % NL], ((nl / NL) - 1) & 1u)) issue_load(nl++);
      if (ns < pick.nb && mbar_try_wait(&sfull[ns % NS], (ns / NS) & 1u)) {
        const unsigned long long row = rowq[ns % kStRows];
        const uint64_t sp = snake && ns + a.keep >= nb_static ? pol_keep : pol;
        bulk_s2g(gbase + row_of_batch(row) * a.pitch, smem + (NL + ns % NS) * a.buf_stride, row_bytes, sp);
        bulk_commit();
        if (ns >= 1) {  // the previous store has left its slot
          bulk_wait_read<1>();
          mbar_arrive(&sfree[(ns - 1) % NS]);
        }
        ++ns;
      }
      if (loads_done && ns >= pick.nb) break;
    }
    bulk_wait<0>();  // every store landed before the CTA retires
    if (a.dbg) {
      a.dbg[kDbg * cta] = smid();
      a.dbg[kDbg * cta + 1] = pick.nb;
      a.dbg[kDbg * cta + 2] = t_start;
      a.dbg[kDbg * cta + 3] = static_cast<unsigned>(globaltimer_ns());
    }
    return;
  }

  if (warp > NW) {
    // ====================================================== factor warps ==
    // alpha_i = rescale_factor(rpd_i, s_i, fi) (fused.hpp:133), batches round
    // robin over the NF warps; sentinel batches publish alpha < 0.
    const unsigned f = static_cast<unsigned>(warp - NW - 1);
    const unsigned long long tag_hi = static_cast<unsigned long long>(ctl->epoch) << 32;
    double errmax = 0.0;
    for (unsigned s = f;; s += NF) {
      const unsigned q = s % kStQ;
      mbar_wait(&done1[q], (s / kStQ) & 1u);
      const unsigned long long packed = rowq[s % kStRows];
      if (packed == kNoRow) {
        if (lane == 0) {
          alpha_s[q] = -1.0;
          mbar_arrive(&alpha_rdy[q]);
        }
        break;
      }
      const unsigned long long row = row_of_batch(packed);
      const double rv = __ldg(&a.rpd[row]);
      double t = red[q * NW2];  // this CTA's partial of the row, warp order
#pragma unroll
      for (int w = 1; w < NW2; ++w) t += red[q * NW2 + w];
      if (XCHG) t = exchange_row_sum(a.xrec, cta, group, G, s % kRing, tag_hi | (s + 1), t, ctl);
      double al = 0.0;
      if (!rescale_factor_dev(rv, t, a.fi, &al)) {
        atomicOr(&ctl->alpha_bad, 1);
        al = 1.0;
      }
      if (g == 0) {
        if (lane == 0) a.alpha[row] = al;
        errmax = fmax(errmax, fabs(al - 1.0));
      }
      if (lane == 0) {
        alpha_s[q] = al;
        mbar_arrive(&alpha_rdy[q]);
      }
    }
    if (lane == 0) {
      a.cta_err[kErrSlots * cta + f] = errmax;
      if (f == 0)
        for (int k = NF; k < kErrSlots; ++k) a.cta_err[kErrSlots * cta + k] = 0.0;
    }
    return;
  }

  // ========================================================= compute warps ==
  const bool sweep1_role = tid < NT2;
  const unsigned t = sweep1_role ? tid : tid - NT2;
  const unsigned w = t >> 5;  // partner warps w (sweep 1) and NW2 + w (sweep 2) share lanes and columns
  const uint32_t lanes = static_cast<uint32_t>(32 * (w % 4)) << 16;
  const uint32_t fcol = tbase + lanes + 8 * V2 * (w / 4);                   // + 8k: factors of chunk k
  const uint32_t xcol = tbase + lanes + FCOLS + 4 * V2 * (w / 4);           // + RCOLS*j + 4k: x1 of chunk k, slot j
  if (sweep1_role) {
    ScreenBounds sb;
    {
      double beta[4 * V2];
      const double* bsrc = a.beta2 + ((ctl->iter + 1) & 1ull) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
      for (int k = 0; k < V2; ++k) {
        const unsigned q = t + k * NT2;
#pragma unroll
        for (int e = 0; e < 4; ++e) beta[4 * k + e] = (FULL || q < nq) ? bsrc[4 * q + e] : 1.0;
      }
      sb = screen_bounds(beta, 4 * V2);
#pragma unroll
      for (int k = 0; k < V2; ++k) tmem_st_chunk(fcol + 8 * k, beta + 4 * k);
      tmem_wait_st_();
    }
    for (unsigned s = 0;; ++s) {
      const unsigned slot = s % NL;
      mbar_wait(&full[slot], (s / NL) & 1u);
      if (rowq[s % kStRows] == kNoRow) {  // no batch left: release the factor warps' sentinels
        if (lane == 0)
          for (int i = 0; i < NF; ++i) mbar_arrive(&done1[(s + i) % kStQ]);
        break;
      }
      const unsigned j = s % NTM;
      if (s >= static_cast<unsigned>(NTM)) {
        mbar_wait(&tfree[j], ((s / NTM) - 1) & 1u);  // sweep 2 has read batch s - NTM from slot j
        tmem_fence_after_();
      }
      const float4* row = reinterpret_cast<const float4*>(smem + slot * a.buf_stride);
      bool bad = false;
      double sacc[4];
#pragma unroll
      for (int g0 = 0; g0 < V2; g0 += KG) {
        double bq[4 * KG];
#pragma unroll
        for (int kk = 0; kk < KG; ++kk) tmem_ld_chunk(fcol + 8 * (g0 + kk), bq + 4 * kk);
        float4 v[KG];
        load_group<NT2, KG, FULL>(row, v, g0, t, nq);
        const uint32_t m = screen_group<KG>(v, sb.lo);
        tmem_wait_ld_();
        double tt[4];
        if (m <= sb.span) {
#pragma unroll
          for (int kk = 0; kk < KG; ++kk)
#pragma unroll
            for (int e = 0; e < 4; ++e) comp(v[kk], e) = d2f(fastd(comp(v[kk], e)) * bq[4 * kk + e]);
#pragma unroll
          for (int e = 0; e < 4; ++e) tt[e] = (FULL || t + g0 * NT2 < nq) ? fastd(comp(v[0], e)) : 0.0;
#pragma unroll
          for (int kk = 1; kk < KG; ++kk)
            if (FULL || t + (g0 + kk) * NT2 < nq)
#pragma unroll
              for (int e = 0; e < 4; ++e) tt[e] += fastd(comp(v[kk], e));
        } else {  // exact hardware conversions for any input
          bad = true;
#pragma unroll
          for (int kk = 0; kk < KG; ++kk)
#pragma unroll
            for (int e = 0; e < 4; ++e)
              comp(v[kk], e) = d2f(static_cast<double>(comp(v[kk], e)) * bq[4 * kk + e]);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            tt[e] = (FULL || t + g0 * NT2 < nq) ? static_cast<double>(comp(v[0], e)) : 0.0;
#pragma unroll
          for (int kk = 1; kk < KG; ++kk)
            if (FULL || t + (g0 + kk) * NT2 < nq)
#pragma unroll
              for (int e = 0; e < 4; ++e) tt[e] += static_cast<double>(comp(v[kk], e));
        }
        tmem_st_x8f(xcol + RCOLS * j + 4 * g0, v[0], v[1]);
#pragma unroll
        for (int e = 0; e < 4; ++e) sacc[e] = g0 == 0 ? tt[e] : sacc[e] + tt[e];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&lfree[slot]);  // every read of the load slot is done
      const double ts = warp_sum((sacc[0] + sacc[1]) + (sacc[2] + sacc[3]));
      const unsigned any_bad = __any_sync(0xffffffffu, bad);
      const unsigned q = s % kStQ;
      if (lane == 0) {
        red[q * NW2 + w] = ts;
        xbad[q * NW2 + w] = any_bad;
      }
      tmem_wait_st_();
      tmem_fence_before_();
      __syncwarp();
      if (lane == 0) mbar_arrive(&done1[q]);
    }
  } else {
    double acc[4 * V2];
#pragma unroll
    for (int i = 0; i < 4 * V2; ++i) acc[i] = 0.0;
    for (unsigned b = 0;; ++b) {
      const unsigned q = b % kStQ;
      mbar_wait(&alpha_rdy[q], (b / kStQ) & 1u);
      const double al = alpha_s[q];
      if (al < 0.0) break;
      tmem_fence_after_();
      const unsigned j = b % NTM, so = b % NS;
      const bool exact = xbad[q * NW2 + w] != 0u || !(al >= 1.0 / kAlphaMargin && al <= kAlphaMargin);
      if (b >= static_cast<unsigned>(NS)) mbar_wait(&sfree[so], ((b / NS) - 1) & 1u);
      float4* out = reinterpret_cast<float4*>(smem + (NL + so) * a.buf_stride);
      // x1 in halves of the row (two chunk groups per tcgen05.wait::ld): the
      // 4*V2 column partials already hold 8*V2 registers
      constexpr int H = UOT_STAGED_H;
#pragma unroll
      for (int h0 = 0; h0 < V2; h0 += H) {
        float4 x[H];
#pragma unroll
        for (int g0 = 0; g0 < H; g0 += KG) tmem_ld_x8f(xcol + RCOLS * j + 4 * (h0 + g0), x[g0], x[g0 + 1]);
        tmem_wait_ld_();
        if (h0 + H >= V2) {  // every x1 of the row is in registers: the TMEM row slot is free for batch b + NTM
          tmem_fence_before_();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tfree[j]);
        }
#pragma unroll
        for (int g0 = 0; g0 < H; g0 += KG) {
          float4 wv[KG] = {x[g0], x[g0 + 1]};
          if (exact)
            group_sweep2<NT2, KG, FULL, true>(out, wv, h0 + g0, t, nq, al, acc);
          else
            group_sweep2<NT2, KG, FULL, false>(out, wv, h0 + g0, t, nq, al, acc);
        }
      }
      fence_proxy_async_smem();  // generic writes -> the producer's bulk store
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[so]);
    }
    double* dst = a.partials + static_cast<size_t>(group) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
    for (int k = 0; k < V2; ++k) {
      const unsigned q = t + k * NT2;
      if (q < nq) {
        reinterpret_cast<double2*>(dst)[2 * q] = make_double2(acc[4 * k], acc[4 * k + 1]);
        reinterpret_cast<double2*>(dst)[2 * q + 1] = make_double2(acc[4 * k + 2], acc[4 * k + 3]);
      }
    }
  }
  // both roles are done with TMEM: compute warp 0 frees it
  tmem_fence_before_();
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  if (warp == 0) {
    tmem_fence_after_();
    tmem_dealloc_cols<512>(tbase);
  }
}

}  // namespace uotk
