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
//   * Warp-specialised: NW compute warps + 1 control warp. The control warp
//     streams rows through a ring of NBUF shared-memory slots with 1-D bulk
//     copies (TMA engine, UBLKCP) signalled on mbarriers, L batches ahead,
//     derives the row factors, and stores finished rows back with bulk
//     shared->global copies. Both sweeps run out of shared memory in place, so
//     P is read from and written to HBM exactly once per iteration.
//   * Compute warps never meet a CTA-wide barrier: they hand batches to the
//     control warp through mbarriers (done1: row partials written; done2: sweep
//     2 finished) and wait only for the data (full) and the factors (alpha_rdy),
//     which the control warp produces one batch ahead of need.
//   * Per-column state lives in registers of the owning thread: beta_j (f64)
//     and the column partial next_j (f64). Thread t owns float4 chunks
//     t, t+NT, ... of the slice (conflict-free 128-bit smem access).
//   * Row sums: thread partial -> warp xor-tree -> per-warp smem -> control
//     lane sums the NW warp partials in warp order. With G > 1 the G CTA
//     partials of a row are exchanged through L2 as 128-bit single-copy-atomic
//     {value, tag} records (no fences) with an LA-batch lag that hides the
//     round trip, then summed in ascending g, so every CTA of the group derives
//     the bit-identical alpha_i. No float atomics; deterministic run to run.
//   * Arithmetic is exactly the reference's: f64 products rounded once to fp32
//     (F2F.F32.F64), f64 sums of the stored fp32 values. f32->f64 uses a
//     two-integer-op conversion with an exact out-of-line fallback.
#pragma once
#include <cstdint>

#include "ptx.cuh"
#include "uot_device.cuh"

namespace uotk {

struct SweepArgs {
  float* P;                   // [rows][pitch] fp32, device layout
  const double* beta2;        // [2][pitch] column factors; beta(t) lives in slot t&1
  const double* rpd;          // [rows] row marginals
  double* alpha;              // [rows] row factors (output)
  double* partials;           // [groups][pitch] column partials (output)
  double* cta_err;            // [grid] max|alpha-1| seen by each CTA (output)
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
  double fi;
};

constexpr int kRing = 8;   // exchange records per CTA
constexpr int kQ = 4;      // ring depth of row partials / factors handed between roles

struct D4 {
  double a, b, c, d;
};

// Exact hardware conversion, out of line so the fast path stays branch-only.
__device__ __noinline__ D4 cvt4_slow(float4 v) { return D4{v.x, v.y, v.z, v.w}; }

// f64 of four stored fp32 values. Fast path: all four positive normal
// (exponent rebias + mantissa shift, two integer ops each).
__device__ __forceinline__ D4 cvt4(float4 v) {
  const uint32_t u0 = __float_as_uint(v.x), u1 = __float_as_uint(v.y);
  const uint32_t u2 = __float_as_uint(v.z), u3 = __float_as_uint(v.w);
  const uint32_t m = max(max(max(u0 - 0x800000u, u1 - 0x800000u), u2 - 0x800000u), u3 - 0x800000u);
  D4 o{__hiloint2double(static_cast<int>((u0 >> 3) + 0x38000000u), static_cast<int>(u0 << 29)),
       __hiloint2double(static_cast<int>((u1 >> 3) + 0x38000000u), static_cast<int>(u1 << 29)),
       __hiloint2double(static_cast<int>((u2 >> 3) + 0x38000000u), static_cast<int>(u2 << 29)),
       __hiloint2double(static_cast<int>((u3 >> 3) + 0x38000000u), static_cast<int>(u3 << 29))};
  if (__builtin_expect(m >= 0x7f000000u, 0)) o = cvt4_slow(v);
  return o;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // xor tree: every lane holds the bit-identical total (fp add commutes)
}

// Shared-memory layout shared by host sizing and the kernel.
template <int NW, int BM, int NBUF>
struct SweepSmem {
  static constexpr int kBars = NBUF /*full*/ + NBUF /*done2*/ + kQ /*done1*/ + kQ /*alpha_rdy*/;
  static constexpr int kDoubles = kQ * NW * BM /*red*/ + kQ * BM /*alpha*/;
  static size_t bytes(unsigned buf_stride) {
    return static_cast<size_t>(NBUF) * buf_stride + kBars * 8 + kDoubles * 8;
  }
};

// NT compute threads (+32 control), V float4 chunks per thread per row
// (slice <= 4*NT*V), BM max rows per batch, NBUF ring slots, XCHG: G > 1
// (cross-CTA row-sum exchange), SEED: the read-only init_col_sums sweep.
template <int NT, int V, int BM, int NBUF, bool XCHG, bool SEED>
__global__ void __launch_bounds__(NT + 32, 1) sweep_kernel(const SweepArgs a) {
  constexpr int NW = NT / 32;
  constexpr int LA = XCHG ? 1 : 0;  // extra batches until a row factor is known
  // ring: L loading + batch in sweep 1 + LA waiting + batch in sweep 2 + one storing
  constexpr int L = SEED ? NBUF : NBUF - LA - 3;
  constexpr int STORE_SLACK = NBUF - L - LA - 2;  // stores issued after the slot's last one
  static_assert(L >= 1 && (SEED || STORE_SLACK >= 0), "ring too small");
  static_assert(!XCHG || BM == 1, "the exchange path moves one row per batch");
  using Smem = SweepSmem<NW, BM, NBUF>;

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
  uint64_t* alpha_rdy = done1 + kQ;
  double* red = reinterpret_cast<double*>(alpha_rdy + kQ);  // [kQ][NW][BM]
  double* alpha_s = red + kQ * NW * BM;                      // [kQ][BM]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned G = a.G;
  const unsigned group = blockIdx.x / G, g = blockIdx.x % G;
  // balanced_blocks over groups (plan.cpp:11-21): first rows%groups get one more.
  const unsigned long long base = a.rows / a.groups, rem = a.rows % a.groups;
  const unsigned long long r0 = group * base + (group < rem ? group : rem);
  const unsigned nrows = static_cast<unsigned>(base + (group < rem ? 1 : 0));
  const unsigned B = a.B;
  const unsigned nb = (nrows + B - 1) / B;
  const unsigned nq = a.slice >> 2;
  const uint32_t row_bytes = a.slice * 4u;
  float* gbase = a.P + r0 * a.pitch + static_cast<size_t>(g) * a.slice;

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
  }
  __syncthreads();

  auto slot_ptr = [&](unsigned b) -> float* {
    return reinterpret_cast<float*>(smem + (b % NBUF) * a.buf_stride);
  };
  auto rows_in = [&](unsigned b) -> unsigned { return min(B, nrows - b * B); };

  if (warp == NW) {
    // ======================================================= control warp ==
    const uint64_t pol = a.evict_first ? policy_evict_first() : policy_evict_normal();
    auto issue_load = [&](unsigned b) {
      const unsigned nr = rows_in(b);
      uint64_t* bar = &full[b % NBUF];
      float* dst = slot_ptr(b);
      const float* src = gbase + static_cast<size_t>(b) * B * a.pitch;
      mbar_arrive_expect_tx(bar, nr * row_bytes);
      if (G == 1) {
        bulk_g2s(dst, src, nr * row_bytes, bar, pol);  // rows contiguous when G == 1
      } else {
        for (unsigned r = 0; r < nr; ++r)
          bulk_g2s(dst + r * a.slice, src + static_cast<size_t>(r) * a.pitch, row_bytes, bar, pol);
      }
    };
    auto issue_store = [&](unsigned b) {
      const unsigned nr = rows_in(b);
      const float* srcs = slot_ptr(b);
      float* dst = gbase + static_cast<size_t>(b) * B * a.pitch;
      if (G == 1) {
        bulk_s2g(dst, srcs, nr * row_bytes, pol);
      } else {
        for (unsigned r = 0; r < nr; ++r)
          bulk_s2g(dst + static_cast<size_t>(r) * a.pitch, srcs + r * a.slice, row_bytes, pol);
      }
      bulk_commit();
    };

    if (lane == 0)
      for (unsigned b = 0; b < nb && b < static_cast<unsigned>(L); ++b) issue_load(b);

    if (SEED) {
      // The compute warps release a slot (done2) as soon as they accumulated it.
      for (unsigned b = NBUF; b < nb; ++b) {
        mbar_wait(&done2[(b - NBUF) % NBUF], ((b - NBUF) / NBUF) & 1u);
        if (lane == 0) issue_load(b);
        __syncwarp();
      }
      return;
    }

    const unsigned long long tag_hi = static_cast<unsigned long long>(ctl->epoch) << 32;
    double errmax = 0.0;
    for (unsigned s = 0; s < nb + LA + 2; ++s) {
      // (a) row factors of batch s (G == 1) or the CTA partial of batch s (G > 1).
      if (s < nb) {
        const unsigned nr = rows_in(s);
        const unsigned q = s % kQ;
        double rv = 0.0;
        if (lane < static_cast<int>(nr)) rv = __ldg(&a.rpd[r0 + static_cast<unsigned long long>(s) * B + lane]);
        mbar_wait(&done1[q], (s / kQ) & 1u);
        if (lane < static_cast<int>(nr)) {
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) t += red[(q * NW + w) * BM + lane];  // warp order
          if (!XCHG) {
            double al;
            if (!rescale_factor_dev(rv, t, a.fi, &al)) {
              atomicOr(&ctl->alpha_bad, 1);
              al = 1.0;
            }
            alpha_s[q * BM + lane] = al;
            a.alpha[r0 + static_cast<unsigned long long>(s) * B + lane] = al;
            errmax = fmax(errmax, fabs(al - 1.0));
          } else {
            st_relaxed_b128(&a.xrec[static_cast<size_t>(blockIdx.x) * kRing + (s % kRing)],
                            static_cast<unsigned long long>(__double_as_longlong(t)), tag_hi | (s + 1));
          }
        }
        if (!XCHG) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&alpha_rdy[q]);
        }
      }
      // (b) G > 1: gather batch s-1 from the G CTAs of the group (published a
      //     batch ago), sum in ascending g, derive its factor.
      if (XCHG && s >= 1 && s - 1 < nb) {
        const unsigned sp = s - 1;
        const unsigned q = sp % kQ;
        double rv = 0.0, v = 0.0;
        if (lane == 0) rv = __ldg(&a.rpd[r0 + sp]);
        if (lane < static_cast<int>(G)) {
          const ulonglong2* rec = &a.xrec[static_cast<size_t>(group * G + lane) * kRing + (sp % kRing)];
          const unsigned long long want = tag_hi | (sp + 1);
          unsigned long long lo, hi;
          ld_relaxed_b128(rec, lo, hi);
          if (hi != want) {
            const unsigned long long t0 = globaltimer_ns();
            do {
              __nanosleep(64);
              ld_relaxed_b128(rec, lo, hi);
              if (hi != want && globaltimer_ns() - t0 > kExchangeTimeoutNs) {
                atomicOr(&ctl->status, kStatusExchangeTimeout);
                break;
              }
            } while (hi != want);
          }
          v = __longlong_as_double(static_cast<long long>(lo));
        }
        double tot = 0.0;
        for (unsigned k = 0; k < G; ++k) tot += __shfl_sync(0xffffffffu, v, k);
        if (lane == 0) {
          double al;
          if (!rescale_factor_dev(rv, tot, a.fi, &al)) {
            atomicOr(&ctl->alpha_bad, 1);
            al = 1.0;
          }
          alpha_s[q * BM] = al;
          if (g == 0) {
            a.alpha[r0 + sp] = al;
            errmax = fmax(errmax, fabs(al - 1.0));
          }
          mbar_arrive(&alpha_rdy[q]);
        }
        __syncwarp();
      }
      // (c) store the batch whose sweep 2 finished (compute step s-1), then
      //     refill the ring: the slot of batch s+L last held batch s+L-NBUF,
      //     whose store left STORE_SLACK stores ago.
      if (s >= static_cast<unsigned>(LA + 2) && s - (LA + 2) < nb) {
        const unsigned b = s - (LA + 2);
        mbar_wait(&done2[b % NBUF], (b / NBUF) & 1u);
        if (lane == 0) issue_store(b);
      }
      if (s + L < nb && lane == 0) {
        bulk_wait_read<STORE_SLACK>();
        issue_load(s + L);
      }
      __syncwarp();
    }
    if (lane == 0) bulk_wait<0>();  // every store landed before the CTA retires
    for (int o = 16; o > 0; o >>= 1) errmax = fmax(errmax, __shfl_xor_sync(0xffffffffu, errmax, o));
    if (lane == 0) a.cta_err[blockIdx.x] = errmax;
    return;
  }

  // ========================================================= compute warps ==
  double beta[4 * V], acc[4 * V];
#pragma unroll
  for (int i = 0; i < 4 * V; ++i) acc[i] = 0.0;
  if (!SEED) {
    const double* bsrc = a.beta2 + ((ctl->iter + 1) & 1ull) * a.pitch + static_cast<size_t>(g) * a.slice;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const unsigned q = tid + k * NT;
#pragma unroll
      for (int e = 0; e < 4; ++e) beta[4 * k + e] = q < nq ? bsrc[4 * q + e] : 0.0;
    }
  }

  const unsigned nsteps = SEED ? nb : nb + LA + 1;
  for (unsigned s = 0; s < nsteps; ++s) {
    // sweep 1 on batch s (or the seed accumulation).
    if (s < nb) {
      mbar_wait(&full[s % NBUF], (s / NBUF) & 1u);
      float* buf = slot_ptr(s);
      const unsigned nr = rows_in(s);
      if (SEED) {
#pragma unroll
        for (int r = 0; r < BM; ++r) {
          if (r < static_cast<int>(nr)) {
            const float4* row = reinterpret_cast<const float4*>(buf + r * a.slice);
#pragma unroll
            for (int k = 0; k < V; ++k) {
              const unsigned q = tid + k * NT;
              if (q < nq) {
                const D4 d = cvt4(row[q]);
                acc[4 * k + 0] += d.a;
                acc[4 * k + 1] += d.b;
                acc[4 * k + 2] += d.c;
                acc[4 * k + 3] += d.d;
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&done2[s % NBUF]);
        continue;
      }
      double part[BM];
#pragma unroll
      for (int r = 0; r < BM; ++r) {
        part[r] = 0.0;
        if (r < static_cast<int>(nr)) {
          float4* row = reinterpret_cast<float4*>(buf + r * a.slice);
          double sr = 0.0;
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const unsigned q = tid + k * NT;
            if (q < nq) {
              float4 v = row[q];
              const D4 d = cvt4(v);
              v.x = d2f(d.a * beta[4 * k + 0]);
              v.y = d2f(d.b * beta[4 * k + 1]);
              v.z = d2f(d.c * beta[4 * k + 2]);
              v.w = d2f(d.d * beta[4 * k + 3]);
              const D4 x1 = cvt4(v);
              sr = sr + x1.a + x1.b + x1.c + x1.d;
              row[q] = v;
            }
          }
          part[r] = sr;
        }
      }
      const unsigned qq = s % kQ;
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

    // sweep 2 on batch s-1-LA once its factors are published.
    if (!SEED && s >= static_cast<unsigned>(LA + 1) && s - (LA + 1) < nb) {
      const unsigned b = s - (LA + 1);
      const unsigned qb = b % kQ;
      mbar_wait(&alpha_rdy[qb], (b / kQ) & 1u);
      float* buf = slot_ptr(b);
      const unsigned nr = rows_in(b);
#pragma unroll
      for (int r = 0; r < BM; ++r) {
        if (r < static_cast<int>(nr)) {
          const double al = alpha_s[qb * BM + r];
          float4* row = reinterpret_cast<float4*>(buf + r * a.slice);
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const unsigned q = tid + k * NT;
            if (q < nq) {
              float4 v = row[q];
              const D4 d = cvt4(v);
              v.x = d2f(d.a * al);
              v.y = d2f(d.b * al);
              v.z = d2f(d.c * al);
              v.w = d2f(d.d * al);
              const D4 x2 = cvt4(v);
              acc[4 * k + 0] += x2.a;
              acc[4 * k + 1] += x2.b;
              acc[4 * k + 2] += x2.c;
              acc[4 * k + 3] += x2.d;
              row[q] = v;
            }
          }
        }
      }
      fence_proxy_async_smem();  // generic writes -> the control warp's bulk store
      __syncwarp();
      if (lane == 0) mbar_arrive(&done2[b % NBUF]);
    }
  }

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
