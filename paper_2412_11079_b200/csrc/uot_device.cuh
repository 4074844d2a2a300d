// uot_device.cuh — device-resident solver state and the scalar factor math.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace uotk {

constexpr int kStatusDegenerateAlpha = 1;   // rescale_factor threw for a row (scaling.cpp:15-22)
constexpr int kStatusDegenerateBeta = 2;    // beta_from_state threw (fused.hpp:146-157)
constexpr int kStatusExchangeTimeout = 4;   // a peer CTA never published (co-residency bug)
constexpr int kStatusPeerTimeout = 8;       // a peer rank never published its column sums
constexpr unsigned long long kPeerTimeoutNs = 60000000000ull;
constexpr int kErrSlots = 4;                // max|alpha-1| slots per sweep CTA (one per factor warp)
constexpr unsigned long long kExchangeTimeoutNs = 4000000000ull;

// One per session, in device memory. Written only by kernels between launches
// (and by the host through reset kernels), so every kernel of one iteration sees
// the same flags. The iteration loop of fused_solve (fused.hpp:273-281) lives
// here: `iter` counts completed iterations, `done` stops the remaining queued
// kernels once the error crossed tol or a factor degenerated.
struct Control {
  unsigned long long iter;    // completed iterations since the problem was set
  unsigned long long epoch;   // never reset: tags of the cross-CTA exchange
  unsigned long long xseq;    // never reset: completed cross-rank exchanges (peer flags)
  unsigned long long allreduce_calls;   // CommStats (distributed.hpp:24-27)
  unsigned long long doubles_reduced;
  double tol;
  double last_error;          // convergence_error of the last completed iteration
  double err_beta[2];         // max|beta(t)-1| at slot t&1 (max on the bit pattern)
  int done;
  int converged;
  int status;                 // sticky kStatus* bits
  int beta_bad;               // beta of the next sweep is degenerate
  int beta_bad_next;          // being produced by the running finalize
  int alpha_bad;              // a row factor of the running sweep degenerated
  unsigned int fin_count;     // last-block election in finalize
  unsigned int bar_count;     // grid barrier of the resident kernel (arrivals)
  unsigned int bar_gen;       // grid barrier generation (never reset)
  unsigned int pad_;
  double rerr_beta[3];        // resident kernel: max|beta(t)-1| at slot t%3
  double rerr_alpha[3];       // resident kernel: max|alpha(t)-1| at slot t%3
  unsigned long long batch_next;  // dynamic sweep: next batch to hand out (0 between sweeps)
  unsigned long long sweep_seq;   // never reset: completed sweep + finalize pairs (mail tags)
  double fin_alpha_err;           // single-rank finalize: block 0's max|alpha-1| for the last block
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// rescale_factor (src/scaling.cpp:15-22): (target/sum)^fi, sum > 0, result
// positive and finite. Returns false where the reference throws DegenerateSum.
__device__ __forceinline__ bool rescale_factor_dev(double target, double sum, double fi,
                                                   double* out) {
  if (!(sum > 0.0)) return false;
  const double f = pow(target / sum, fi);
  if (!(f > 0.0) || !isfinite(f)) return false;
  *out = f;
  return true;
}

// max on non-negative doubles through their (monotone) bit patterns.
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace uotk
