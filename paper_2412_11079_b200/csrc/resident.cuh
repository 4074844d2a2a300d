// resident.cuh — K fused iterations in ONE persistent kernel, the matrix
// resident in shared memory (small problems: BASELINE configs 1 and the like).
//
// When a CTA's row block fits in shared memory (rows/grid x pitch x 4 bytes <=
// ~200 KB, e.g. 1024 x 1024 on 148 SMs: 7 rows x 4 KB), streaming it from HBM
// every iteration and relaunching sweep + finalize costs far more than the
// arithmetic: the iteration becomes launch- and latency-bound (sweep.cuh +
// finalize.cuh: ~35 us per 1024^2 iteration). Here one cooperative launch keeps
// every CTA's rows in shared memory for all K iterations and replaces the
// finalize kernel with two grid barriers per iteration:
//
//   sweep 1 of all resident rows (fused.hpp:125-131)      -> row partials
//   alpha_i = rescale_factor(rpd_i, s_i, fi)              (fused.hpp:133)
//   sweep 2 of all resident rows (fused.hpp:135-142)      -> column partials
//   ---- grid barrier ----
//   CTA c: columns [c*cpc, (c+1)*cpc): next_j = sum_k partial_k[j] in ascending
//   k (fused.hpp:242-248), beta_j(t+1) (fused.hpp:146-157), max|beta-1|
//   ---- grid barrier ----
//   every CTA: error(t) = max(max|alpha-1|, max|beta(t)-1|) (scaling.cpp:24-29)
//   from the same global values -> the same stop decision (fused.hpp:277-280)
//
// The per-element arithmetic is the streaming kernel's (row_sweep1/row_sweep2
// of sweep.cuh), so results agree with it to the summation order of the f64
// row/column sums (both within 1e-16 relative of each other, both exact
// products). P is read from and written to HBM once per SOLVE, not per
// iteration.
#pragma once
#include "sweep.cuh"

namespace uotk {

struct ResidentArgs {
  float* P;                // [rows][pitch]
  double* beta2;           // [2][pitch]; beta(t) in slot t&1
  const double* rpd;       // [rows]
  const double* cpd;       // [cols]
  double* alpha;           // [rows] factors of the last completed iteration
  double* partials;        // [grid][pitch] column partials of the running iteration
  double* col_sums;        // [cols] carried FusedState::col_sums
  unsigned* bar_flags;     // [grid] arrival epochs of the grid barrier (zeroed once per session)
  Control* ctl;
  unsigned long long rows;
  unsigned int cols, pitch, grid;
  unsigned int k;          // iterations requested by this launch
  double fi;
};

// Grid barrier over the co-resident CTAs of a cooperative launch, without
// atomics: CTA c publishes the barrier's epoch in its own flag (release), then
// thread t of every CTA waits for flag t (acquire) — one L2 round trip after
// the last arrival instead of nblocks serialised atomics on one address.
// Epochs grow monotonically across launches (Control::bar_gen).
#ifdef UOT_FLAG_BARRIER
__device__ __forceinline__ void grid_barrier(unsigned* flags, Control*, unsigned nblocks, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_u32(&flags[blockIdx.x], epoch);
  for (unsigned t = threadIdx.x; t < nblocks; t += blockDim.x)
    while (static_cast<int>(ld_acquire_u32(&flags[t]) - epoch) < 0) {
    }
  __syncthreads();
}
#else
// One arrival counter per barrier instance: the last CTA to arrive publishes the
// epoch, the others spin on it (one thread per CTA).
__device__ __forceinline__ void grid_barrier(unsigned* flags, Control* ctl, unsigned nblocks, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&flags[epoch & 1u], 1u) == nblocks - 1) {
      flags[epoch & 1u] = 0;  // reused two barriers later: every CTA has left this one by then
      st_release_u32(&ctl->bar_gen, epoch);
    } else {
      while (static_cast<int>(ld_acquire_u32(&ctl->bar_gen) - epoch) < 0) {
      }
    }
  }
  __syncthreads();
}
#endif

template <int NT, int V>
struct ResidentSmem {
  // rows x pitch floats, then red[NW][rows] and alpha[rows] doubles
  static size_t bytes(unsigned rows_cta, unsigned pitch) {
    const size_t m = static_cast<size_t>(rows_cta) * pitch * 4;
    return (m + 15) / 16 * 16 + static_cast<size_t>(NT / 32 + 1) * rows_cta * 8;
  }
};

// trace build: CTA 0 thread 0 times the phases of each iteration into uot_trace[24..29]
#ifdef UOT_TRACE
#define RT_MARK(id)                                                              \
  do {                                                                           \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                   \
      const unsigned long long now_ = clock64();                                 \
      atomicAdd(&uot_trace[id], now_ - rt_t);                                    \
      rt_t = now_;                                                               \
    }                                                                            \
  } while (0)
#else
#define RT_MARK(id)
#endif

template <int NT, int V, bool FULL>
__global__ void __launch_bounds__(NT, 1) resident_kernel(const ResidentArgs a) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  Control* ctl = a.ctl;
  if (ctl->done) return;
  const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned c = blockIdx.x;
  const unsigned long long base = a.rows / a.grid, rem = a.rows % a.grid;  // plan.cpp:11-21
  const unsigned long long r0 = c * base + (c < rem ? c : rem);
  const unsigned nr = static_cast<unsigned>(base + (c < rem ? 1 : 0));
  const unsigned rmax = static_cast<unsigned>(base + (rem ? 1 : 0));
  const unsigned nq = a.pitch >> 2;
  float* rows = reinterpret_cast<float*>(smem);
  double* red = reinterpret_cast<double*>(smem + (static_cast<size_t>(rmax) * a.pitch * 4 + 15) / 16 * 16);
  double* alpha_s = red + NW * rmax;

  // the row block: HBM -> shared memory, once per solve
  {
    const float4* src = reinterpret_cast<const float4*>(a.P + r0 * a.pitch);
    float4* dst = reinterpret_cast<float4*>(rows);
    for (unsigned i = tid; i < nr * nq; i += NT) dst[i] = src[i];
  }
  __syncthreads();

  const unsigned long long t0 = ctl->iter;  // completed iterations before this launch
  const double tol = ctl->tol;
  // error slots: beta(t0+1)'s max|beta-1| was produced by the finalize before us
  if (c == 0 && tid == 0) {
    ctl->rerr_beta[(t0 + 1) % 3] = ctl->err_beta[(t0 + 1) & 1ull];
    ctl->rerr_beta[(t0 + 2) % 3] = 0.0;
    ctl->rerr_alpha[(t0 + 1) % 3] = 0.0;
    ctl->rerr_alpha[(t0 + 2) % 3] = 0.0;
  }
  bool beta_bad = ctl->beta_bad != 0;
  unsigned epoch = *reinterpret_cast<volatile unsigned*>(&ctl->bar_gen);  // advanced only by the barriers
  grid_barrier(a.bar_flags, ctl, a.grid, ++epoch);

  double beta[4 * V];
  unsigned long long t = t0;  // completed iterations
  double err = ctl->last_error;
  bool stop = false, conv = false, adeg = false;
#ifdef UOT_TRACE
  unsigned long long rt_t = clock64();
#endif
  for (unsigned it = 0; it < a.k && !stop; ++it) {
    const unsigned long long tt = t + 1;  // the iteration running now
    if (beta_bad) {  // beta_from_state threw at the top of iteration tt (fused.hpp:146-157)
      if (c == 0 && tid == 0) atomicOr(&ctl->status, kStatusDegenerateBeta);
      break;
    }
    const double* bsrc = a.beta2 + (tt & 1ull) * a.pitch;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = tid + k * NT;
#pragma unroll
      for (int e = 0; e < 4; ++e) beta[4 * k + e] = (FULL || q < nq) ? __ldcg(&bsrc[4 * q + e]) : 1.0;
    }
    const ScreenBounds sb = screen_bounds(beta, 4 * V);
    RT_MARK(24);

    // ---- sweep 1 of every resident row, row partials in warp order
    uint32_t bad_rows = 0;  // rows_cta <= 32 for the eligible shapes (host-checked)
    for (unsigned r = 0; r < nr; ++r) {
      bool bad = false;
      const double p = row_sweep1<NT, V, FULL>(reinterpret_cast<float4*>(rows + static_cast<size_t>(r) * a.pitch),
                                               tid, nq, beta, sb, bad);
      if (bad) bad_rows |= 1u << r;
      const double w = warp_sum(p);
      if (lane == 0) red[warp * rmax + r] = w;
    }
    __syncthreads();
    RT_MARK(25);
    // ---- row factors: thread r sums the NW warp partials of row r in order
    double aerr = 0.0;
    for (unsigned r = tid; r < nr; r += NT) {
      double s = red[r];
      for (int w = 1; w < NW; ++w) s += red[w * rmax + r];
      double al;
      if (!rescale_factor_dev(__ldg(&a.rpd[r0 + r]), s, a.fi, &al)) {
        atomicOr(&ctl->alpha_bad, 1);
        al = 1.0;
      }
      alpha_s[r] = al;
      a.alpha[r0 + r] = al;
      aerr = fmax(aerr, fabs(al - 1.0));
    }
    __syncthreads();
    RT_MARK(26);
    // ---- sweep 2, column partials of this CTA in registers
    double acc[4 * V];
#pragma unroll
    for (int i = 0; i < 4 * V; ++i) acc[i] = 0.0;
    for (unsigned r = 0; r < nr; ++r)
      row_sweep2<NT, V, FULL>(reinterpret_cast<float4*>(rows + static_cast<size_t>(r) * a.pitch), tid, nq,
                              alpha_s[r], (bad_rows >> r) & 1u, acc);
    double* dst = a.partials + static_cast<size_t>(c) * a.pitch;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = tid + k * NT;
      if (q < nq) {
        reinterpret_cast<double2*>(dst)[2 * q] = make_double2(acc[4 * k + 0], acc[4 * k + 1]);
        reinterpret_cast<double2*>(dst)[2 * q + 1] = make_double2(acc[4 * k + 2], acc[4 * k + 3]);
      }
    }
    // alpha error of this iteration: global max (slot tt % 3)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) aerr = fmax(aerr, __shfl_xor_sync(0xffffffffu, aerr, o));
    if (lane == 0 && aerr > 0.0) atomic_max_nonneg(&ctl->rerr_alpha[tt % 3], aerr);
    if (c == 0 && tid == 0) {  // slots next accumulated at iteration tt+1, last read at tt-2
      ctl->rerr_alpha[(tt + 1) % 3] = 0.0;
      ctl->rerr_beta[(tt + 1) % 3] = 0.0;
    }
    RT_MARK(27);
    grid_barrier(a.bar_flags, ctl, a.grid, ++epoch);
    RT_MARK(28);

    // ---- column reduction: warp w of CTA c takes columns c*cpc + w, + NW, ...;
    // lane l loads partials l, l+32, ... (all in flight at once), adds them in
    // ascending order, then the xor tree: a fixed order, deterministic.
    const unsigned cpc = (a.pitch + a.grid - 1) / a.grid;
    double berr = 0.0;
    for (unsigned jj = warp; jj < cpc; jj += NW) {
      const unsigned j = c * cpc + jj;
      if (j >= a.pitch) break;
      constexpr int kMaxK = 8;  // grid <= 256 CTAs
      double v[kMaxK];
#pragma unroll
      for (int i = 0; i < kMaxK; ++i) {
        const unsigned k = lane + 32u * i;
        v[i] = k < a.grid ? __ldcg(&a.partials[static_cast<size_t>(k) * a.pitch + j]) : 0.0;
      }
      double s = v[0];
#pragma unroll
      for (int i = 1; i < kMaxK; ++i) s += v[i];
      s = warp_sum(s);
      if (lane == 0) {
        double b = 0.0;
        if (j < a.cols) {
          a.col_sums[j] = s;
          if (!rescale_factor_dev(a.cpd[j], s, a.fi, &b)) {
            ctl->beta_bad_next = 1;
            b = 1.0;
          }
          berr = fmax(berr, fabs(b - 1.0));
        }
        a.beta2[((tt + 1) & 1ull) * a.pitch + j] = b;  // padding columns: 0
      }
    }
    if (lane == 0 && berr > 0.0) atomic_max_nonneg(&ctl->rerr_beta[(tt + 1) % 3], berr);
    RT_MARK(29);
    grid_barrier(a.bar_flags, ctl, a.grid, ++epoch);
    RT_MARK(30);

    // ---- the stop test from the same global values on every CTA
    const double ea = *reinterpret_cast<volatile double*>(&ctl->rerr_alpha[tt % 3]);
    const double eb = *reinterpret_cast<volatile double*>(&ctl->rerr_beta[tt % 3]);
    if (*reinterpret_cast<volatile int*>(&ctl->alpha_bad)) {  // a row pass threw: tt did not complete
      adeg = true;
      break;
    }
    t = tt;
    err = fmax(ea, eb);
    beta_bad = *reinterpret_cast<volatile int*>(&ctl->beta_bad_next) != 0;
    if (err <= tol) {
      conv = true;
      stop = true;
    }
  }
  __syncthreads();

  // the row block back to HBM
  {
    float4* dst = reinterpret_cast<float4*>(a.P + r0 * a.pitch);
    const float4* src = reinterpret_cast<const float4*>(rows);
    for (unsigned i = tid; i < nr * nq; i += NT) dst[i] = src[i];
  }
  grid_barrier(a.bar_flags, ctl, a.grid, ++epoch);  // every CTA read the flags before CTA 0 rewrites them
  if (c == 0 && tid == 0) {
    if (adeg) ctl->status |= kStatusDegenerateAlpha;
    if (ctl->status) ctl->done = 1;
    ctl->epoch += t - t0;
    ctl->iter = t;
    ctl->last_error = err;
    if (conv) {
      ctl->converged = 1;
      ctl->done = 1;
    }
    ctl->beta_bad = beta_bad ? 1 : 0;
    ctl->beta_bad_next = 0;
    // hand the error slot of beta(t+1) back to the streaming path's parity slots
    ctl->err_beta[(t + 1) & 1ull] = ctl->rerr_beta[(t + 1) % 3];
    ctl->err_beta[t & 1ull] = 0.0;
  }
}

}  // namespace uotk
