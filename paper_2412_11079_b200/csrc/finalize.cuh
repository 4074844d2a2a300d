// finalize.cuh — the O(cols) tail of an iteration, one small kernel.
//
//   next[j] = sum_k partial_k[j]                     fused.hpp:242-248 (ordered reduction)
//   beta_j  = rescale_factor(cpd_j, next[j], fi)     fused.hpp:146-157, scaling.cpp:15-22
//   error   = max(max_i|alpha_i-1|, max_j|beta_j-1|) scaling.cpp:24-29; stop test fused.hpp:277-280
//
// The reference derives beta at the top of iteration t+1; here the tail of
// iteration t computes it eagerly into the other parity slot (beta(t) stays
// readable as the factor set of iteration t). A degenerate beta(t+1) is only
// raised when a next sweep actually runs (sweep_kernel reads beta_bad), exactly
// where the reference would throw.
//
// Layout: a block owns kFinCols consecutive columns; its 8 warps split the
// `groups` partial rows by k mod 8 (each warp reads 32 consecutive doubles per
// row: 256-byte coalesced) and warp 0 adds the 8 slice sums in slice order. The
// summation order is fixed, so results are deterministic run to run; the
// latency chain per thread is groups/8 loads instead of groups.
//
// Multi-GPU (distributed.hpp:88-100), one exchange of the column sums per
// iteration, two ways (XCH):
//   kXchNccl  stage 1 writes this rank's column sums into the allreduce vector
//             (plus its alpha error in slot cols+rank), the host enqueues one
//             ncclAllReduce(sum), stage 2 consumes the result.
//   kXchPeer  the allreduce fused into the two stages over peer memory (CUDA
//             IPC, NVLink/NVSwitch): stage 1 PUSHES this rank's column sums and
//             alpha error into row `rank` of every peer's receive table with
//             plain remote stores, then its last block raises a sequence flag in
//             every peer (st.release.sys); stage 2 waits for all P flags in its
//             own memory and sums the P rows in ascending rank order — exactly
//             allreduce_vectors (src/allreduce.cpp:6-15), identical bits on every
//             rank, no NCCL launch. Receive tables are double-buffered by the
//             parity of the exchange sequence number (a rank can be at most one
//             exchange ahead of any peer).
#pragma once
#include "ptx.cuh"
#include "uot_device.cuh"

namespace uotk {

constexpr int kFinThreads = 256;
constexpr int kFinSlices = kFinThreads / 32;
constexpr int kFinCols = 32;

enum XchMode : int { kXchNone = 0, kXchNccl = 1, kXchPeer = 2 };

// Per-rank peer-exchange region (identical layout on every rank):
//   u64    flags[2][nranks]           sequence number of the last exchange seen per sender
//   double recv[2][nranks][xlen]      row q = rank q's column sums, then its alpha error
struct PeerRegion {
  __host__ __device__ static size_t flag_bytes(unsigned nranks) { return (2ull * nranks * 8 + 255) / 256 * 256; }
  static size_t bytes(unsigned nranks, unsigned xlen) {
    return flag_bytes(nranks) + 2ull * nranks * xlen * sizeof(double);
  }
};

struct FinalizeArgs {
  const double* partials;  // [groups][pitch]
  const double* cta_err;   // [grid][kErrSlots]
  const double* cpd;       // [cols]
  double* beta2;           // [2][pitch]
  double* col_sums;        // [cols]  carried FusedState::col_sums
  double* xsum;            // [cols + nranks] allreduce vector (kXchNccl) or nullptr
  unsigned char* const* peers;  // [nranks] peer-region base of every rank (kXchPeer; own included)
  unsigned char* region;        // this rank's peer region (kXchPeer)
  Control* ctl;
  unsigned int cols, pitch, groups, grid, rank, nranks, xlen;
  double fi;
};

enum FinalizeMode : int {
  kFinSeed = 0,      // after the init_col_sums sweep: next -> col_sums -> beta(1)
  kFinIter = 1,      // after an iteration sweep: col_sums, beta(t+1), error(t), stop test
  kFinBetaOnly = 2,  // col_sums uploaded by the host (FusedState given) -> beta(iter+1)
};

// max over the sweep CTAs' alpha errors, by the whole block (result in every thread).
__device__ __forceinline__ double block_alpha_err(const FinalizeArgs& f, double* red) {
  double e = 0.0;
  for (unsigned c = threadIdx.x; c < kErrSlots * f.grid; c += kFinThreads) e = fmax(e, f.cta_err[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  double m = 0.0;
#pragma unroll
  for (int w = 0; w < kFinSlices; ++w) m = fmax(m, red[w]);
  __syncthreads();
  return m;
}

__device__ __forceinline__ unsigned long long* peer_flags(unsigned char* base) {
  return reinterpret_cast<unsigned long long*>(base);
}
__device__ __forceinline__ double* peer_recv(unsigned char* base, unsigned nranks) {
  return reinterpret_cast<double*>(base + PeerRegion::flag_bytes(nranks));
}

// R > 0: every thread issues its R partial-row loads at once (groups <= 8R);
// R = 0: batches of 8 (any number of groups). R sets the register footprint, so
// the launch picks the smallest that covers the groups (one wave of blocks).
template <int MODE, bool REDUCE, bool BETA, int XCH = kXchNone, int R = 0>
__global__ void __launch_bounds__(kFinThreads) finalize_kernel(const FinalizeArgs f) {
  __shared__ double part[kFinSlices][kFinCols];
  __shared__ double red[kFinSlices];
  __shared__ int last;
  Control* ctl = f.ctl;
  if (ctl->done) return;
  const unsigned lane = threadIdx.x & 31, slice = threadIdx.x >> 5;
  const unsigned j = blockIdx.x * kFinCols + lane;
  const unsigned long long it = ctl->iter;  // completed before this sweep
  const unsigned long long seq = ctl->xseq + 1;  // this exchange (kXchPeer)
  const unsigned par = static_cast<unsigned>(seq & 1ull);

  // The alpha error of a single-rank iteration: block 0 reduces the sweep CTAs'
  // slots while the column loads of every block are in flight, and hands the
  // max to the last block through the control block (published before block
  // 0's election increment), so the last block's tail is only the stop test.
  if (REDUCE && BETA && MODE == kFinIter && blockIdx.x == 0) {
    const double ea = block_alpha_err(f, red);
    if (threadIdx.x == 0) ctl->fin_alpha_err = ea;
  }

  double s = 0.0;  // column sum of column j (valid in warp 0)
  if (REDUCE) {
    // Same ascending-k order of additions as a plain loop, with every L2 load
    // of the thread's rows (k = slice, slice + 8, ...) issued before the first
    // add: one round trip instead of one per batch of rows (a serial loop paid
    // one per row: 13 us at 148 groups).
    double p = 0.0;
    if (j < f.cols) {
      if (R > 0) {
        double v[R > 0 ? R : 1];
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const unsigned k = slice + u * kFinSlices;
          v[u] = k < f.groups ? __ldcg(&f.partials[static_cast<size_t>(k) * f.pitch + j]) : 0.0;
        }
        p = v[0];
#pragma unroll
        for (int u = 1; u < R; ++u)
          if (slice + u * kFinSlices < f.groups) p += v[u];
      } else {
        unsigned k = slice;
        for (; k + 7 * kFinSlices < f.groups; k += 8 * kFinSlices) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            v[u] = __ldcg(&f.partials[static_cast<size_t>(k + u * kFinSlices) * f.pitch + j]);
#pragma unroll
          for (int u = 0; u < 8; ++u) p += v[u];
        }
        for (; k < f.groups; k += kFinSlices) p += __ldcg(&f.partials[static_cast<size_t>(k) * f.pitch + j]);
      }
    }
    part[slice][lane] = p;
    __syncthreads();
    if (slice == 0) {
#pragma unroll
      for (int w = 0; w < kFinSlices; ++w) s += part[w][lane];
    }
  }

  if (REDUCE && !BETA) {  // multi-GPU stage 1: local partial sums -> the exchange
    // this rank's alpha error; a degenerate row factor travels as -1 so every
    // rank stops at the same iteration
    double e = 0.0;
    if (blockIdx.x == 0 && MODE == kFinIter) {
      e = block_alpha_err(f, red);
      if (ctl->alpha_bad) e = -1.0;
    }
    if (XCH == kXchNccl) {
      if (slice == 0 && j < f.cols) f.xsum[j] = s;
      if (blockIdx.x == 0)
        for (unsigned r = threadIdx.x; r < f.nranks; r += kFinThreads) f.xsum[f.cols + r] = r == f.rank ? e : 0.0;
      return;
    }
    // kXchPeer: warp 0 (it holds the sums) pushes into row `rank` of every
    // peer's receive table: 256-byte coalesced remote stores per peer
    if (slice == 0 && j < f.cols)
      for (unsigned q = 0; q < f.nranks; ++q)
        peer_recv(f.peers[q], f.nranks)[(static_cast<size_t>(par) * f.nranks + f.rank) * f.xlen + j] = s;
    if (blockIdx.x == 0 && threadIdx.x < f.nranks) {
      double* row = peer_recv(f.peers[threadIdx.x], f.nranks) + (static_cast<size_t>(par) * f.nranks + f.rank) * f.xlen;
      row[f.cols] = e;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&ctl->fin_count, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence_system();
    if (threadIdx.x < f.nranks) st_release_sys_u64(&peer_flags(f.peers[threadIdx.x])[par * f.nranks + f.rank], seq);
    if (threadIdx.x == 0) ctl->fin_count = 0;
    return;
  }

  if (XCH == kXchPeer && !REDUCE && MODE != kFinBetaOnly) {
    // stage 2: wait until every rank's row of this exchange has landed here
    if (threadIdx.x < f.nranks) {
      const unsigned long long* flag = &peer_flags(f.region)[par * f.nranks + threadIdx.x];
      if (ld_acquire_sys_u64(flag) != seq) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys_u64(flag) != seq) {
          if (globaltimer_ns() - t0 > kPeerTimeoutNs) {
            atomicOr(&ctl->status, kStatusPeerTimeout);
            ctl->done = 1;
            break;
          }
        }
      }
    }
    __syncthreads();
  }

  // beta slot: seed produces beta(1); iteration t = it+1 produces beta(t+1).
  const unsigned long long tb = (MODE == kFinIter) ? it + 2 : it + 1;
  if (slice == 0) {
    double e = 0.0;
    if (j < f.cols) {
      if (MODE == kFinBetaOnly) {
        s = f.col_sums[j];
      } else if (!REDUCE && XCH == kXchPeer) {
        const double* recv = peer_recv(f.region, f.nranks) + static_cast<size_t>(par) * f.nranks * f.xlen;
        s = 0.0;
        for (unsigned q = 0; q < f.nranks; ++q) s += __ldcg(&recv[static_cast<size_t>(q) * f.xlen + j]);
      } else if (!REDUCE) {
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
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
    if (lane == 0) {  // block max -> err_beta slot of beta(tb), then the last-block election
      atomic_max_nonneg(&ctl->err_beta[tb & 1ull], e);
      __threadfence();
      last = atomicAdd(&ctl->fin_count, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;

  // ---- last block: the scalar tail of the iteration ----
  __threadfence();
  double ea = 0.0;
  if (MODE == kFinIter) {
    if (REDUCE) {
      ea = *reinterpret_cast<volatile double*>(&ctl->fin_alpha_err);  // block 0's reduction
    } else if (XCH == kXchPeer) {
      const double* recv = peer_recv(f.region, f.nranks) + static_cast<size_t>(par) * f.nranks * f.xlen;
      for (unsigned q = 0; q < f.nranks; ++q) {
        const double v = __ldcg(&recv[static_cast<size_t>(q) * f.xlen + f.cols]);
        ea = v < 0.0 || ea < 0.0 ? -1.0 : fmax(ea, v);
      }
    } else {
      for (unsigned r = 0; r < f.nranks; ++r) {
        const double v = f.xsum[f.cols + r];
        ea = v < 0.0 || ea < 0.0 ? -1.0 : fmax(ea, v);
      }
    }
  }
  if (threadIdx.x != 0) return;
  ctl->fin_count = 0;
  ctl->batch_next = 0;  // the sweep before this finalize has retired
  ctl->sweep_seq += 1;
  if (XCH != kXchNone && !REDUCE && MODE != kFinBetaOnly) ctl->xseq = seq;
  ctl->beta_bad = ctl->beta_bad_next;
  ctl->beta_bad_next = 0;
  if (MODE == kFinIter) {
    const unsigned long long t = it + 1;
    volatile double* eb = &ctl->err_beta[t & 1ull];
    const double err = fmax(ea, *eb);
    *eb = 0.0;  // this slot next receives beta(t+2)
    if (ctl->alpha_bad || ea < 0.0) {  // a row pass threw: iteration t did not complete
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

inline unsigned finalize_blocks(unsigned pitch) { return (pitch + kFinCols - 1) / kFinCols; }

}  // namespace uotk
