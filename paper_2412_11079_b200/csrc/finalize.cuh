// finalize.cuh — the O(cols) tail of an iteration, one small kernel.
//
//   next[j] = sum_k partial_k[j], k ascending       fused.hpp:242-248 (worker order)
//   beta_j  = rescale_factor(cpd_j, next[j], fi)     fused.hpp:146-157, scaling.cpp:15-22
//   error   = max(max_i|alpha_i-1|, max_j|beta_j-1|) scaling.cpp:24-29; stop test fused.hpp:277-280
//
// The reference derives beta at the top of iteration t+1; here the tail of
// iteration t computes it eagerly into the other parity slot (beta(t) stays
// readable as the factor set of iteration t). A degenerate beta(t+1) is only
// raised when a next sweep actually runs (sweep_kernel reads beta_bad), exactly
// where the reference would throw.
//
// Multi-GPU (distributed.hpp:88-100): REDUCE writes this rank's column partial
// sum into the exchange vector (plus its alpha-error in slot cols+rank), the
// host enqueues one ncclAllReduce(sum) on it, and BETA consumes the result.
#pragma once
#include "uot_device.cuh"

namespace uotk {

struct FinalizeArgs {
  const double* partials;  // [groups][pitch]
  const double* cta_err;   // [grid][2]
  const double* cpd;       // [cols]
  double* beta2;           // [2][pitch]
  double* col_sums;        // [cols]  carried FusedState::col_sums
  double* xsum;            // [cols + nranks] allreduce vector (multi-GPU) or nullptr
  Control* ctl;
  unsigned int cols, pitch, groups, grid, rank, nranks;
  double fi;
};

enum FinalizeMode : int {
  kFinSeed = 0,      // after the init_col_sums sweep: next -> col_sums -> beta(1)
  kFinIter = 1,      // after an iteration sweep: col_sums, beta(t+1), error(t), stop test
  kFinBetaOnly = 2,  // col_sums uploaded by the host (FusedState given) -> beta(iter+1)
};

template <int MODE, bool REDUCE, bool BETA>
__global__ void __launch_bounds__(256) finalize_kernel(const FinalizeArgs f) {
  Control* ctl = f.ctl;
  if (ctl->done) return;
  const unsigned j = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long it = ctl->iter;  // completed before this sweep

  if (REDUCE && !BETA) {  // multi-GPU stage 1: local partial sums -> exchange vector
    if (j < f.cols) {
      double s = 0.0;
      for (unsigned k = 0; k < f.groups; ++k) s += f.partials[static_cast<size_t>(k) * f.pitch + j];
      f.xsum[j] = s;
    }
    if (j < f.nranks) {  // this rank's alpha error in its own slot, zeros elsewhere
      double e = 0.0;
      if (j == f.rank && MODE == kFinIter)
        for (unsigned c = 0; c < 2 * f.grid; ++c) e = fmax(e, f.cta_err[c]);
      f.xsum[f.cols + j] = e;
    }
    return;
  }

  // beta slot: seed produces beta(1); iteration t = it+1 produces beta(t+1).
  const unsigned long long tb = (MODE == kFinIter) ? it + 2 : it + 1;
  double e = 0.0;
  if (j < f.cols) {
    double s;
    if (MODE == kFinBetaOnly) {
      s = f.col_sums[j];
    } else if (REDUCE) {
      s = 0.0;
      for (unsigned k = 0; k < f.groups; ++k) s += f.partials[static_cast<size_t>(k) * f.pitch + j];
    } else {
      s = f.xsum[j];  // allreduced
    }
    if (MODE != kFinBetaOnly) f.col_sums[j] = s;
    double b;
    if (!rescale_factor_dev(f.cpd[j], s, f.fi, &b)) {
      ctl->beta_bad_next = 1;
      b = 1.0;
    }
    f.beta2[(tb & 1ull) * f.pitch + j] = b;
    e = fabs(b - 1.0);
  } else if (j < f.pitch) {
    f.beta2[(tb & 1ull) * f.pitch + j] = 0.0;  // padding columns hold zeros in P
  }
  // block max -> err_beta slot of beta(tb)
  __shared__ double wmax[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < 8; ++w) m = fmax(m, wmax[w]);
    atomic_max_nonneg(&ctl->err_beta[tb & 1ull], m);
    __threadfence();
    const unsigned done_blocks = atomicAdd(&ctl->fin_count, 1u);
    if (done_blocks == gridDim.x - 1) {  // last block: the scalar tail
      __threadfence();
      ctl->fin_count = 0;
      ctl->beta_bad = ctl->beta_bad_next;
      ctl->beta_bad_next = 0;
      if (MODE == kFinIter) {
        const unsigned long long t = it + 1;
        double ea = 0.0;
        if (REDUCE) {
          for (unsigned c = 0; c < 2 * f.grid; ++c) ea = fmax(ea, f.cta_err[c]);
        } else {
          for (unsigned r = 0; r < f.nranks; ++r) ea = fmax(ea, f.xsum[f.cols + r]);
        }
        volatile double* eb = &ctl->err_beta[t & 1ull];
        const double err = fmax(ea, *eb);
        *eb = 0.0;  // this slot next receives beta(t+2)
        if (ctl->alpha_bad) {  // the row pass threw: iteration t did not complete
          ctl->status |= kStatusDegenerateAlpha;
          ctl->done = 1;
        } else {
          ctl->iter = t;
          ctl->last_error = err;
          if (err <= ctl->tol) {
            ctl->converged = 1;
            ctl->done = 1;
          }
        }
        ctl->epoch += 1;
      }
    }
  }
}

}  // namespace uotk
