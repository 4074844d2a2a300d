// ablation.cuh — the two unfused iteration schedules the paper compares the
// fused sweep against, as plain sm_100a streaming kernels:
//
//   TWO_PASS  the paper's GPU data flow (tiled.hpp:210-229): part4 applies the
//             column factors and accumulates row sums (one read + one write of
//             P), the row factors follow, part2 applies them and accumulates
//             column sums (another read + write): 16 B per fp32 element.
//   BASELINE  the reference's four-sweep iteration (baseline.hpp:100-110):
//             column sums (read), column scaling (read + write), row sums
//             (read), row scaling (read + write): 24 B per element, the
//             metrics.cpp:60-77 model (4 loads + 2 stores per element).
//
// The fused sweep (sweep.cuh) moves 8 B per element. These kernels exist to
// measure the bytes-per-iteration claim on real HBM; they compute the same
// iteration (identical products, f64 sums in a different order), so their plans
// agree with the oracle to the parity bar. Row kernels give each row to one
// warp (coalesced 512-byte float4 runs); column kernels give each thread V
// float4 column chunks of a row block and keep the f64 column partials in
// registers, written to a [row blocks][pitch] table the finalize kernel reduces.
#pragma once
#include <type_traits>

#include "sweep.cuh"

namespace uotk {

constexpr int kAblRowWarps = 8;  // rows (warps) per CTA of the row kernels
constexpr int kAblColThreads = 256;
constexpr int kAblColV = 4;      // float4 chunks per thread: 4096 columns per CTA

struct AblArgs {
  void* P;               // [rows][pitch] float (Problem<float>) or double (Problem<double>)
  const double* beta2;   // [2][pitch]
  const double* rpd;
  double* alpha;
  double* partials;      // [gy][pitch]
  double* row_err;       // [row CTAs] max|alpha-1| per row CTA (zero padded)
  Control* ctl;
  unsigned long long rows;
  unsigned int cols, pitch, gy;
  double fi;
};

// x (f32) widened exactly: two integer ops for positive normal values, the
// hardware conversion otherwise (one screen per float4).
__device__ __forceinline__ void widen4(float4 v, double (&d)[4]) {
  uint32_t m = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) m = nn_max(m, comp(v, e));
  if (nn_ok(m)) {
#pragma unroll
    for (int e = 0; e < 4; ++e) d[e] = fastd(comp(v, e));
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) d[e] = static_cast<double>(comp(v, e));
  }
}

__device__ __forceinline__ bool abl_stopped(Control* ctl, bool check_beta) {
  if (ctl->done) return true;
  if (check_beta && ctl->beta_bad) {  // beta_from_state threw (fused.hpp:146-157)
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
      atomicOr(&ctl->status, kStatusDegenerateBeta);
      ctl->done = 1;
    }
    return true;
  }
  return false;
}

// One warp per row. SCALE_BETA: x <- f32(f64(x)*beta_j) first (part4). SUM:
// s = sum_j f64(x) -> alpha_i = rescale_factor(rpd_i, s, fi) (fused.hpp:133 /
// baseline.hpp:65-76). SCALE_ALPHA: x <- f32(f64(x)*alpha_i) (baseline row
// scaling, baseline.hpp:78-88).
// T = double (Problem<double>): the same schedule on plain f64 products, one
// element per lane step (the f64 ablations exist for parity / verify).
template <bool SCALE_BETA, bool SUM, bool SCALE_ALPHA, typename T = float>
__global__ void __launch_bounds__(32 * kAblRowWarps) abl_row_kernel(const AblArgs a) {
  Control* ctl = a.ctl;
  if (abl_stopped(ctl, SCALE_BETA)) return;
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * kAblRowWarps + w;
  __shared__ double werr[kAblRowWarps];
  double err = 0.0;
  if (i < a.rows) {
    const double* beta = a.beta2 + ((ctl->iter + 1) & 1ull) * a.pitch;
    double s = 0.0;
    double al = SCALE_ALPHA ? a.alpha[i] : 1.0;
    if constexpr (std::is_same<T, double>::value) {
      double* row = static_cast<double*>(a.P) + i * a.pitch;
      for (unsigned j = lane; j < a.cols; j += 32) {
        double x = row[j];
        if (SCALE_BETA) x *= beta[j];
        if (SCALE_ALPHA) x *= al;
        if (SCALE_BETA || SCALE_ALPHA) row[j] = x;
        if (SUM) s += x;
      }
    } else {
    float4* row = reinterpret_cast<float4*>(static_cast<float*>(a.P) + i * a.pitch);
    const unsigned nq = (a.cols + 3) / 4;
    for (unsigned q = lane; q < nq; q += 32) {
      float4 v = row[q];
      double d[4];
      widen4(v, d);
      if (SCALE_BETA) {
#pragma unroll
        for (int e = 0; e < 4; ++e) comp(v, e) = d2f(d[e] * beta[4 * q + e]);
        widen4(v, d);
      }
      if (SCALE_ALPHA) {
#pragma unroll
        for (int e = 0; e < 4; ++e) comp(v, e) = d2f(d[e] * al);
      }
      if (SCALE_BETA || SCALE_ALPHA) row[q] = v;
      if (SUM) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * q + e < a.cols) s += d[e];
      }
    }
    }
    if (SUM) {
      s = warp_sum(s);
      if (lane == 0) {
        if (!rescale_factor_dev(a.rpd[i], s, a.fi, &al)) {
          atomicOr(&ctl->alpha_bad, 1);
          al = 1.0;
        }
        a.alpha[i] = al;
        err = fabs(al - 1.0);
      }
    }
  }
  if (SUM) {
    if (lane == 0) werr[w] = err;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int k = 0; k < kAblRowWarps; ++k) m = fmax(m, werr[k]);
      a.row_err[blockIdx.x] = m;
    }
  }
}

// Column kernel over a row block: grid (gx column tiles, gy row blocks).
// SCALE_ALPHA: x <- f32(f64(x)*alpha_i) first (part2). SCALE_BETA: x <-
// f32(f64(x)*beta_j) (baseline column scaling, baseline.hpp:48-56). SUM: column
// partials of the (scaled) values -> partials[by][j] (baseline.hpp:30-38 /
// fused.hpp:135-142).
template <bool SCALE_ALPHA, bool SCALE_BETA, bool SUM, typename T = float>
__global__ void __launch_bounds__(kAblColThreads) abl_col_kernel(const AblArgs a) {
  Control* ctl = a.ctl;
  if (abl_stopped(ctl, SCALE_BETA)) return;
  constexpr int V = kAblColV;
  const unsigned nq = a.pitch / 4;
  const unsigned q0 = blockIdx.x * (kAblColThreads * V) + threadIdx.x;
  const unsigned long long base = a.rows / a.gy, rem = a.rows % a.gy;  // plan.cpp:11-21
  const unsigned by = blockIdx.y;
  const unsigned long long r0 = by * base + (by < rem ? by : rem);
  const unsigned long long r1 = r0 + base + (by < rem ? 1 : 0);
  double acc[4 * V], beta[4 * V];
#pragma unroll
  for (int k = 0; k < 4 * V; ++k) acc[k] = 0.0;
  if (SCALE_BETA) {
    const double* b = a.beta2 + ((ctl->iter + 1) & 1ull) * a.pitch;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = q0 + k * kAblColThreads;
#pragma unroll
      for (int e = 0; e < 4; ++e) beta[4 * k + e] = 4 * q + e < a.pitch ? b[4 * q + e] : 0.0;
    }
  }
  if constexpr (std::is_same<T, double>::value) {  // 4 scalar columns per chunk, bounds per element
    for (unsigned long long i = r0; i < r1; ++i) {
      double* row = static_cast<double*>(a.P) + i * a.pitch;
      const double al = SCALE_ALPHA ? a.alpha[i] : 1.0;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const unsigned q = q0 + k * kAblColThreads;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const unsigned j = 4 * q + e;
          if (j < a.pitch) {
            double x = row[j];
            if (SCALE_ALPHA || SCALE_BETA) {
              x *= SCALE_ALPHA ? al : beta[4 * k + e];
              row[j] = x;
            }
            if (SUM) acc[4 * k + e] += x;
          }
        }
      }
    }
    if (SUM) {
      double* dst = a.partials + static_cast<size_t>(by) * a.pitch;
#pragma unroll
      for (int k = 0; k < V; ++k)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const unsigned j = 4 * (q0 + k * kAblColThreads) + e;
          if (j < a.pitch) dst[j] = acc[4 * k + e];
        }
    }
    return;
  }
  for (unsigned long long i = r0; i < r1; ++i) {
    float4* row = reinterpret_cast<float4*>(static_cast<float*>(a.P) + i * a.pitch);
    const double al = SCALE_ALPHA ? a.alpha[i] : 1.0;
    float4 v[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = q0 + k * kAblColThreads;
      v[k] = q < nq ? row[q] : make_float4(1.f, 1.f, 1.f, 1.f);
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = q0 + k * kAblColThreads;
      double d[4];
      widen4(v[k], d);
      if (SCALE_ALPHA || SCALE_BETA) {
#pragma unroll
        for (int e = 0; e < 4; ++e) comp(v[k], e) = d2f(d[e] * (SCALE_ALPHA ? al : beta[4 * k + e]));
        if (q < nq) row[q] = v[k];
        if (SUM) widen4(v[k], d);
      }
      if (SUM && q < nq) {
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[4 * k + e] += d[e];
      }
    }
  }
  if (SUM) {
    double* dst = a.partials + static_cast<size_t>(by) * a.pitch;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = q0 + k * kAblColThreads;
      if (q < nq) {
        reinterpret_cast<double2*>(dst)[2 * q] = make_double2(acc[4 * k + 0], acc[4 * k + 1]);
        reinterpret_cast<double2*>(dst)[2 * q + 1] = make_double2(acc[4 * k + 2], acc[4 * k + 3]);
      }
    }
  }
}

// End of a baseline iteration t: error(t) = max(max|alpha-1|, max|beta(t)-1|)
// (scaling.cpp:24-29), stop test (baseline.hpp:130-136). beta(t) and its error
// slot were produced by this iteration's column-sum finalize (seed mode).
__global__ void abl_baseline_tail_kernel(const AblArgs a, unsigned nrow_ctas) {
  Control* ctl = a.ctl;
  if (ctl->done) return;
  __shared__ double red[32];
  double e = 0.0;
  for (unsigned c = threadIdx.x; c < nrow_ctas; c += blockDim.x) e = fmax(e, a.row_err[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double ea = 0.0;
  for (unsigned w = 0; w < (blockDim.x + 31) / 32; ++w) ea = fmax(ea, red[w]);
  const unsigned long long t = ctl->iter + 1;
  const double err = fmax(ea, ctl->err_beta[t & 1ull]);
  ctl->err_beta[t & 1ull] = 0.0;
  if (ctl->alpha_bad) {
    ctl->status |= kStatusDegenerateAlpha;
    ctl->done = 1;
    return;
  }
  ctl->iter = t;
  ctl->last_error = err;
  ctl->epoch += 1;
  if (err <= ctl->tol) {
    ctl->converged = 1;
    ctl->done = 1;
  }
}

}  // namespace uotk
