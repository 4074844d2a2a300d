// problem.cuh — device-side problem generation and validation.
//
// gen_problem_t (include/uot/problem_io.hpp:17-31) draws A row-major, then rpd,
// then cpd from ONE SplitMix64 stream (include/uot/rng.hpp:9-25). Draw k only
// depends on seed + (k+1)*gamma, so every element is generated independently
// and the device problem is bit-identical to the host one without a host
// generation pass or an H2D copy of A.
#pragma once
#include <cstdint>

#include "uot_device.cuh"

namespace uotk {

__device__ __forceinline__ double splitmix_unit_at(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return static_cast<double>((z >> 11) + 1) * 0x1p-53;
}

// A (local rows [row0, row0+rows) of a global rows x cols problem) into the
// pitched layout; padding columns are zero. T = float: the draw cast to fp32
// (gen_problem_t<float>), T = double: the draw itself.
template <typename T>
__global__ void gen_matrix_kernel(T* P, uint64_t seed, unsigned long long row0,
                                  unsigned long long rows, unsigned cols, unsigned pitch) {
  const unsigned long long n = rows * pitch;
  for (unsigned long long idx = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
       idx < n; idx += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long i = idx / pitch;
    const unsigned j = static_cast<unsigned>(idx - i * pitch);
    P[idx] = j < cols ? static_cast<T>(splitmix_unit_at(seed, (row0 + i) * cols + j)) : T(0);
  }
}

// rpd (local slice) and cpd: draws after the whole global matrix.
__global__ void gen_marginals_kernel(double* rpd, double* cpd, uint64_t seed,
                                     unsigned long long grows, unsigned long long row0,
                                     unsigned long long rows, unsigned cols) {
  const unsigned long long mn = grows * cols;
  for (unsigned long long k = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
       k < rows + cols; k += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    if (k < rows)
      rpd[k] = splitmix_unit_at(seed, mn + row0 + k);
    else
      cpd[k - rows] = splitmix_unit_at(seed, mn + grows + (k - rows));
  }
}

// validate_problem's matrix rule (include/uot/problem.hpp:85-90): every entry
// strictly positive and finite. Padding columns are skipped. Sets *bad.
template <typename T>
__global__ void validate_matrix_kernel(const T* P, unsigned long long rows, unsigned cols,
                                       unsigned pitch, int* bad) {
  const unsigned long long n = rows * pitch;
  int local = 0;
  for (unsigned long long idx = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
       idx < n; idx += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned j = static_cast<unsigned>(idx % pitch);
    const T v = P[idx];
    if (j < cols && !(v > T(0) && isfinite(v))) local = 1;
  }
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}

// Zero the padding columns [cols, pitch) after a host upload.
template <typename T>
__global__ void zero_padding_kernel(T* P, unsigned long long rows, unsigned cols, unsigned pitch) {
  const unsigned w = pitch - cols;
  const unsigned long long n = rows * w;
  for (unsigned long long idx = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
       idx < n; idx += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long i = idx / w;
    P[i * pitch + cols + (idx - i * w)] = T(0);
  }
}

// Reset the per-problem part of Control (epoch survives: exchange tags stay unique).
__global__ void reset_control_kernel(Control* c) {
  c->iter = 0;
  c->allreduce_calls = 0;
  c->doubles_reduced = 0;
  c->tol = 0.0;
  c->last_error = 0.0;
  c->err_beta[0] = 0.0;
  c->err_beta[1] = 0.0;
  c->done = 0;
  c->converged = 0;
  c->status = 0;
  c->beta_bad = 0;
  c->beta_bad_next = 0;
  c->alpha_bad = 0;
  c->fin_count = 0;
  c->batch_next = 0;
}

// Undo a calibration run (uot_calibrate_schedule): the per-problem fields come
// back from `saved`; the never-reset tags (epoch, xseq, sweep_seq) keep moving
// forward so no stale exchange record or mailbox entry can match again.
__global__ void restore_control_kernel(Control* c, const Control* saved) {
  c->iter = saved->iter;
  c->allreduce_calls = saved->allreduce_calls;
  c->doubles_reduced = saved->doubles_reduced;
  c->tol = saved->tol;
  c->last_error = saved->last_error;
  c->err_beta[0] = saved->err_beta[0];
  c->err_beta[1] = saved->err_beta[1];
  c->done = saved->done;
  c->converged = saved->converged;
  c->status = saved->status;
  c->beta_bad = saved->beta_bad;
  c->beta_bad_next = saved->beta_bad_next;
  c->alpha_bad = saved->alpha_bad;
  c->fin_count = 0;
  c->batch_next = 0;
}

// A caller-supplied FusedState (uot_set_col_sums): a converged session may run
// again; a failed one stays stopped.
__global__ void resume_control_kernel(Control* c) {
  c->converged = 0;
  c->done = c->status != 0 ? 1 : 0;
}

// Start of an iterate() call: new tolerance; a failed session stays stopped.
__global__ void begin_iterate_kernel(Control* c, double tol) {
  c->tol = tol;
  c->converged = 0;
  c->done = c->status != 0 ? 1 : 0;
  c->batch_next = 0;
}

}  // namespace uotk
