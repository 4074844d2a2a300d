// persist.cuh — K fused iterations in ONE persistent streaming launch.
//
// The streaming sweep (sweep.cuh) is launched once per iteration and followed
// by the finalize kernel (finalize.cuh): every iteration drains and refills the
// TMA ring and pays the finalize kernel (~14 us of latency-bound work) plus two
// kernel boundaries. Here the same warp roles loop over all K iterations:
//
//   * the producer warp streams GLOBAL batch indices gb = it*nb + b: as soon as
//     a slot frees near the end of iteration it, it prefetches the first
//     batches of iteration it+1 (loads do not depend on beta), so HBM never
//     idles across iterations;
//   * compute + factor warps finish iteration it, publish the CTA's column
//     partials and max|alpha-1|, and meet the other CTAs at a grid barrier;
//     CTA c then reduces columns [c*cpc, (c+1)*cpc) over the row groups'
//     partials in ascending order (fused.hpp:242-248), derives beta(t+1)
//     (fused.hpp:146-157) and max|beta-1|; after a second grid barrier every CTA
//     evaluates the same stop test (fused.hpp:273-281, scaling.cpp:24-29) from
//     the same global values and either continues with beta(t+1) or stops.
//
// The per-element arithmetic is sweep.cuh's (row_sweep1/row_sweep2), so the plan
// agrees with the per-iteration path up to the summation order of the f64
// column sums. Single rank only (the cross-rank exchange lives in finalize).
// The grid barriers use named barrier 1 (compute + factor warps only: the
// producer keeps streaming meanwhile) around one thread's epoch spin.
#pragma once
#include "sweep.cuh"

namespace uotk {

struct PersistArgs {
  SweepArgs s;
  const double* cpd;
  double* beta2w;      // = s.beta2, writable
  double* col_sums;    // [cols]
  unsigned* bar;       // [2] arrival counters of the grid barrier (zeroed once per session)
  unsigned cols, grid, k;
};

__device__ __forceinline__ void named_barrier(unsigned id, unsigned threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Grid barrier among the participating warps of every CTA: an arrival counter
// per barrier parity; the last arriver publishes the epoch (release), the
// others spin on it (acquire). `threads` = participating threads per CTA.
__device__ __forceinline__ void grid_barrier_part(unsigned* counters, Control* ctl, unsigned nblocks, unsigned epoch,
                                                  unsigned threads, bool leader) {
  named_barrier(1, threads);
  if (leader) {
    __threadfence();
    if (atomicAdd(&counters[epoch & 1u], 1u) == nblocks - 1) {
      counters[epoch & 1u] = 0;  // reused two barriers later: every CTA has left this one by then
      st_release_u32(&ctl->bar_gen, epoch);
    } else {
      while (static_cast<int>(ld_acquire_u32(&ctl->bar_gen) - epoch) < 0) {
      }
    }
    __threadfence();
  }
  named_barrier(1, threads);
}

template <int NT, int V, int BM, int NBUF, int LA, bool XCHG, int NF, bool FULL>
__global__ void __launch_bounds__(NT + 32 * (1 + NF), 1) persist_kernel(const PersistArgs pa) {
  constexpr int NW = NT / 32;
  constexpr unsigned kPart = NT + 32 * NF;  // threads meeting at the grid barriers
  static_assert(NF >= 1 && NF <= kErrSlots, "factor warps");
  static_assert(LA >= 1 && LA <= 2 && (!XCHG || LA == 2), "lag (the alpha / red rings hold kQ batches)");
  static_assert(NBUF >= LA + 4, "ring too small");
  static_assert(!XCHG || BM == 1, "the exchange path moves one row per batch");
  const SweepArgs& a = pa.s;

  extern __shared__ __align__(128) unsigned char smem[];
  Control* ctl = a.ctl;
  if (ctl->done) return;
  if (ctl->beta_bad) {  // beta_from_state throws at the top of the first iteration (fused.hpp:146-157)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(&ctl->status, kStatusDegenerateBeta);
      ctl->done = 1;
    }
    return;
  }

  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NBUF * a.buf_stride);
  uint64_t* done2 = full + NBUF;
  uint64_t* done1 = done2 + NBUF;
  uint64_t* alpha_rdy = done1 + kQ;
  double* red = reinterpret_cast<double*>(alpha_rdy + kQ);  // [kQ][NW][BM]
  double* alpha_s = red + kQ * NW * BM;                      // [kQ][BM]
  __shared__ int stop_flag;
  // iteration-boundary state, owned by thread 0 (kept out of the compute warps'
  // registers: the sweep body is register-bound)
  struct State {
    unsigned long long t, t0, epoch0;
    double err;
    unsigned epoch;
    int conv, adeg, bdeg;
  };
  __shared__ State st;

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
  const unsigned K = pa.k;

  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&done2[i], NW);
    }
    for (int i = 0; i < kQ; ++i) {
      mbar_init(&done1[i], NW);
      mbar_init(&alpha_rdy[i], 1);
    }
    fence_mbar_init();
    stop_flag = 0;
    st.t = st.t0 = ctl->iter;
    st.epoch0 = ctl->epoch;
    st.err = ctl->last_error;
    st.epoch = *reinterpret_cast<volatile unsigned*>(&ctl->bar_gen);
    st.conv = st.adeg = st.bdeg = 0;
  }
  __syncthreads();

  auto slot_ptr = [&](unsigned gb) -> float* {
    return reinterpret_cast<float*>(smem + (gb % NBUF) * a.buf_stride);
  };
  auto rows_in = [&](unsigned b) -> unsigned { return min(B, nrows - b * B); };

  if (warp == NW) {
    // ===================================================== producer warp ==
    if (lane != 0) return;
    const uint64_t pol = a.evict_first ? policy_evict_first() : policy_evict_normal();
    const unsigned total = K * nb;  // host-checked to fit 31 bits
    unsigned next_load = 0;  // global batches issued so far
    auto issue_load = [&](unsigned gb) {
      const unsigned b = static_cast<unsigned>(gb % nb);
      const unsigned nr = rows_in(b);
      uint64_t* bar = &full[gb % NBUF];
      float* dst = slot_ptr(gb);
      const float* src = gbase + static_cast<size_t>(b) * B * a.pitch;
      if (gb >= nb && b < static_cast<unsigned>(NBUF)) {
        // row batch b was stored during the previous iteration: that global
        // write must have landed before the bulk load reads it back
        if (nb > 2u * NBUF)
          bulk_wait<NBUF>();
        else
          bulk_wait<0>();
      }
      mbar_arrive_expect_tx(bar, nr * row_bytes);
      if (G == 1) {
        bulk_g2s(dst, src, nr * row_bytes, bar, pol);
      } else {
        for (unsigned r = 0; r < nr; ++r)
          bulk_g2s(dst + r * a.slice, src + static_cast<size_t>(r) * a.pitch, row_bytes, bar, pol);
      }
      next_load = gb + 1;
    };
    for (unsigned gb = 0; gb < total && gb < static_cast<unsigned>(NBUF); ++gb) issue_load(gb);
    for (unsigned gb = 0; gb < total; ++gb) {
      mbar_wait(&done2[gb % NBUF], (gb / NBUF) & 1u);
      if (*reinterpret_cast<volatile int*>(&stop_flag)) {
        // stopped early: let every issued load land before the CTA retires
        for (unsigned j = gb; j < next_load; ++j) mbar_wait(&full[j % NBUF], (j / NBUF) & 1u);
        break;
      }
      const unsigned b = static_cast<unsigned>(gb % nb);
      const unsigned nr = rows_in(b);
      const float* srcs = slot_ptr(gb);
      float* dst = gbase + static_cast<size_t>(b) * B * a.pitch;
      if (G == 1) {
        bulk_s2g(dst, srcs, nr * row_bytes, pol);
      } else {
        for (unsigned r = 0; r < nr; ++r)
          bulk_s2g(dst + static_cast<size_t>(r) * a.pitch, srcs + r * a.slice, row_bytes, pol);
      }
      bulk_commit();
      if (gb >= 1 && gb - 1 + NBUF < total) {
        bulk_wait_read<1>();
        issue_load(gb - 1 + NBUF);
      }
    }
    bulk_wait<0>();
    return;
  }

  const bool leader = tid == 0;

  if (warp > NW) {
    // ====================================================== factor warps ==
    const unsigned f = static_cast<unsigned>(warp - NW - 1);
    for (unsigned it = 0; it < K; ++it) {
      const unsigned long long tag_hi = (st.epoch0 + it) << 32;
      double errmax = 0.0;
      for (unsigned s = f; s < nb; s += NF) {
        const unsigned gs = it * nb + s;
        const unsigned nr = rows_in(s);
        const unsigned q = gs % kQ;
        double rv = 0.0;
        if (lane < static_cast<int>(nr)) rv = __ldg(&a.rpd[r0 + static_cast<unsigned long long>(s) * B + lane]);
        mbar_wait(&done1[q], (gs / kQ) & 1u);
        double t = 0.0;
        if (lane < static_cast<int>(nr)) {
          t = red[(q * NW) * BM + lane];
#pragma unroll
          for (int w = 1; w < NW; ++w) t += red[(q * NW + w) * BM + lane];
        }
        if (XCHG)  // as sweep.cuh: {partial, tag} records in L2, ascending-g sum
          t = exchange_row_sum(a.xrec, cta, group, G, gs % kRing, tag_hi | (s + 1), t, ctl);

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
      if (lane == 0 && errmax > 0.0) atomic_max_nonneg(&ctl->rerr_alpha[(st.t0 + it + 1) % 3], errmax);
      // the iteration boundary: same barrier sequence as the compute warps
      grid_barrier_part(pa.bar, ctl, pa.grid, 0, kPart, false);
      named_barrier(1, kPart);  // column reduction done in this CTA
      grid_barrier_part(pa.bar, ctl, pa.grid, 0, kPart, false);
      named_barrier(1, kPart);  // stop decision published in smem
      if (stop_flag) return;
    }
    return;
  }

  // ========================================================= compute warps ==
  double beta[4 * V], acc[4 * V];
  if (leader) {  // error slots of this launch (resident.cuh's rotation)
    const unsigned long long t0 = st.t0;
    ctl->rerr_beta[(t0 + 1) % 3] = ctl->err_beta[(t0 + 1) & 1ull];
    ctl->rerr_beta[(t0 + 2) % 3] = 0.0;
    ctl->rerr_alpha[(t0 + 1) % 3] = 0.0;
    ctl->rerr_alpha[(t0 + 2) % 3] = 0.0;
  }
  for (unsigned it = 0; it < K; ++it) {
    const unsigned long long tt = st.t0 + it + 1;  // iterations never resume once stopped
    const double* bsrc = a.beta2 + (tt & 1ull) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = tid + k * NT;
#pragma unroll
      for (int e = 0; e < 4; ++e) beta[4 * k + e] = (FULL || q < nq) ? __ldcg(&bsrc[4 * q + e]) : 1.0;
    }
#pragma unroll
    for (int i = 0; i < 4 * V; ++i) acc[i] = 0.0;
    const ScreenBounds sb = screen_bounds(beta, 4 * V);

    uint64_t x1bad = 0;
    for (unsigned s = 0; s < nb + LA + 1; ++s) {
      const bool s1 = s < nb;
      const bool s2 = s >= static_cast<unsigned>(LA + 1) && s - (LA + 1) < nb;
      const unsigned b = s - (LA + 1);
      const unsigned gs = it * nb + s;
      const unsigned gb2 = it * nb + b;
      double part[BM];
      if (s1) {
        mbar_wait(&full[gs % NBUF], (gs / NBUF) & 1u);
        float* buf = slot_ptr(gs);
        const unsigned nr = rows_in(s);
        const unsigned sh = (s % 8) * 8;
        x1bad &= ~(0xffull << sh);
#pragma unroll
        for (int r = 0; r < BM; ++r) {
          part[r] = 0.0;
          if (r < static_cast<int>(nr)) {
            bool bad = false;
            part[r] = row_sweep1<NT, V, FULL>(reinterpret_cast<float4*>(buf + r * a.slice), tid, nq, beta, sb, bad);
            if (bad) x1bad |= 1ull << (sh + r);
          }
        }
      }
      if (s2) {
        mbar_wait(&alpha_rdy[gb2 % kQ], (gb2 / kQ) & 1u);
        float* buf = slot_ptr(gb2);
        const unsigned nr = rows_in(b);
        const unsigned sh = (b % 8) * 8;
#pragma unroll
        for (int r = 0; r < BM; ++r)
          if (r < static_cast<int>(nr))
            row_sweep2<NT, V, FULL>(reinterpret_cast<float4*>(buf + r * a.slice), tid, nq,
                                    alpha_s[(gb2 % kQ) * BM + r], (x1bad >> (sh + r)) & 1ull, acc);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&done2[gb2 % NBUF]);
      }
      if (s1) {
        const unsigned qq = gs % kQ;
        const unsigned nr = rows_in(s);
#pragma unroll
        for (int r = 0; r < BM; ++r) {
          if (r < static_cast<int>(nr)) {
            const double w = warp_sum(part[r]);
            if (lane == 0) red[(qq * NW + warp) * BM + r] = w;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&done1[qq]);
      }
    }
    // column partials of this CTA for iteration tt
    double* dst = a.partials + static_cast<size_t>(group) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = tid + k * NT;
      if (q < nq) {
        reinterpret_cast<double2*>(dst)[2 * q] = make_double2(acc[4 * k + 0], acc[4 * k + 1]);
        reinterpret_cast<double2*>(dst)[2 * q + 1] = make_double2(acc[4 * k + 2], acc[4 * k + 3]);
      }
    }
    if (leader) {  // slots next accumulated at iteration tt+1, last read at tt-2
      ctl->rerr_alpha[(tt + 1) % 3] = 0.0;
      ctl->rerr_beta[(tt + 1) % 3] = 0.0;
    }
    grid_barrier_part(pa.bar, ctl, pa.grid, leader ? ++st.epoch : 0, kPart, leader);

    // ---- column reduction of this CTA's columns [c*cpc, (c+1)*cpc): a segment
    // of `lpc` lanes per column, lane l of a segment adds partial rows l, l+lpc,
    // ... in ascending order, then an xor tree inside the segment — a fixed
    // order (deterministic) with every thread busy.
    {
      const unsigned cpc = (a.pitch + pa.grid - 1) / pa.grid;
      const unsigned c = blockIdx.x;
      unsigned lpc = 32;
      while (lpc > 1 && lpc * cpc > 32u * NW * 2u) lpc >>= 1;  // lanes per column
      const unsigned cpw = 32 / lpc;                             // columns per warp and round
      const unsigned sl = lane % lpc;
      double berr = 0.0;
      for (unsigned jj0 = warp * cpw; jj0 < cpc; jj0 += NW * cpw) {
        const unsigned jj = jj0 + lane / lpc;
        const unsigned j = c * cpc + jj;
        const bool live = jj < cpc && j < a.pitch;
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        unsigned k = sl;
        if (live) {
          for (; k + 3 * lpc < a.groups; k += 4 * lpc) {  // four loads in flight, added in k order
            const double* col = a.partials + j;
            const double p0 = __ldcg(&col[static_cast<size_t>(k) * a.pitch]);
            const double p1 = __ldcg(&col[static_cast<size_t>(k + lpc) * a.pitch]);
            const double p2 = __ldcg(&col[static_cast<size_t>(k + 2 * lpc) * a.pitch]);
            const double p3 = __ldcg(&col[static_cast<size_t>(k + 3 * lpc) * a.pitch]);
            v0 += p0;
            v0 += p1;
            v0 += p2;
            v0 += p3;
          }
          for (; k < a.groups; k += lpc) v1 += __ldcg(&a.partials[static_cast<size_t>(k) * a.pitch + j]);
        }
        double sum = (v0 + v1) + (v2 + v3);
        for (unsigned o = lpc >> 1; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (live && sl == 0) {
          double bv = 0.0;
          if (j < pa.cols) {
            pa.col_sums[j] = sum;
            if (!rescale_factor_dev(pa.cpd[j], sum, a.fi, &bv)) {
              ctl->beta_bad_next = 1;
              bv = 1.0;
            }
            berr = fmax(berr, fabs(bv - 1.0));
          }
          pa.beta2w[((tt + 1) & 1ull) * a.pitch + j] = bv;  // padding columns: 0
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) berr = fmax(berr, __shfl_xor_sync(0xffffffffu, berr, o));
      if (lane == 0 && berr > 0.0) atomic_max_nonneg(&ctl->rerr_beta[(tt + 1) % 3], berr);
    }
    named_barrier(1, kPart);
    grid_barrier_part(pa.bar, ctl, pa.grid, leader ? ++st.epoch : 0, kPart, leader);

    // ---- the stop test from the same global values on every CTA (thread 0
    // decides; the decision reaches the CTA through shared memory)
    if (leader) {
      const double ea = *reinterpret_cast<volatile double*>(&ctl->rerr_alpha[tt % 3]);
      const double eb = *reinterpret_cast<volatile double*>(&ctl->rerr_beta[tt % 3]);
      int stop = 0;
      if (*reinterpret_cast<volatile int*>(&ctl->alpha_bad)) {  // a row pass threw: tt did not complete
        st.adeg = 1;
        stop = 1;
      } else {
        st.t = tt;
        st.err = fmax(ea, eb);
        st.bdeg = *reinterpret_cast<volatile int*>(&ctl->beta_bad_next) != 0;
        if (st.err <= ctl->tol) {
          st.conv = 1;
          stop = 1;
        }
        if (st.bdeg && it + 1 < K) {  // the next iteration would throw in beta_from_state
          if (blockIdx.x == 0) atomicOr(&ctl->status, kStatusDegenerateBeta);
          stop = 1;
        }
      }
      if (stop) stop_flag = it + 1 < K ? 1 : 2;
    }
    named_barrier(1, kPart);  // stop_flag visible to the compute and factor warps
    const int stop = stop_flag;
    if (stop == 1 && lane == 0)  // release the producer: it waits for sweep 2 of the next iteration's first batch
      mbar_arrive(&done2[((it + 1) * nb) % NBUF]);
    if (stop) break;
  }

  // the final state (every CTA read the flags before the last barrier)
  grid_barrier_part(pa.bar, ctl, pa.grid, leader ? ++st.epoch : 0, NT, leader);  // factor warps have left
  if (blockIdx.x == 0 && leader) {
    const unsigned long long t = st.t;
    if (st.adeg) ctl->status |= kStatusDegenerateAlpha;
    if (ctl->status) ctl->done = 1;
    ctl->epoch = st.epoch0 + K + 1;  // beyond every exchange tag this launch could have used
    ctl->iter = t;
    ctl->last_error = st.err;
    if (st.conv) {
      ctl->converged = 1;
      ctl->done = 1;
    }
    ctl->beta_bad = st.bdeg ? 1 : 0;
    ctl->beta_bad_next = 0;
    ctl->err_beta[(t + 1) & 1ull] = ctl->rerr_beta[(t + 1) % 3];
    ctl->err_beta[t & 1ull] = 0.0;
  }
}

}  // namespace uotk
