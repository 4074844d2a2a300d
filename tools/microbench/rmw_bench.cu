// In-place read-modify-write streaming ceilings on B200 (scratch microbenchmark).
//
// What is the best HBM rate an in-place sweep (read P, write P back) can reach,
// and which mechanism gets there?  Variants over a 4 GiB fp32 buffer:
//   copy_ldg   out-of-place float4 copy (the MEASURED_PEAKS reference pattern)
//   rmw_ldg    in-place float4 x*=c, U loads in flight per thread
//   rmw_bulk   persistent CTA per SM, ring of NS slots of SLOT bytes filled by
//              cp.async.bulk, a consumer warp touching the slot, bulk store back;
//              HOLD extra batches between load completion and store (the
//              sweep's alpha lag); pitch/piece mimic G > 1 row slices.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2412_11079_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace uotk;

__global__ void copy_ldg(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <int U>
__global__ void rmw_ldg(float4* __restrict__ a, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) v[u] = a[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) {
        v[u].x *= 1.0000001f; v[u].y *= 1.0000001f; v[u].z *= 1.0000001f; v[u].w *= 1.0000001f;
        a[i + u * stride] = v[u];
      }
  }
}

// CTA c owns rows [c*rows_per, (c+1)*rows_per) of a [rows][pitch] matrix,
// column piece [g*piece, (g+1)*piece) with g = c % G (G CTAs per row group).
struct BulkArgs {
  float* P;
  size_t rows_per;     // batches per CTA
  unsigned pitch;      // floats
  unsigned piece;      // floats per batch (one row slice)
  unsigned G;
  unsigned hold;       // batches a slot is held after its load lands
  int touch;           // consumer warp reads + writes the slot
  int evict_first;
};

template <int NS>
__global__ void __launch_bounds__(64, 1) rmw_bulk(const BulkArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned bytes = a.piece * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * bytes);
  uint64_t* done = full + NS;
  const unsigned grp = blockIdx.x / a.G, g = blockIdx.x % a.G;
  float* base = a.P + grp * a.rows_per * a.pitch + (size_t)g * a.piece;
  const unsigned nb = a.rows_per;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&done[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane) return;
    const uint64_t pol = a.evict_first ? policy_evict_first() : policy_evict_normal();
    auto load = [&](unsigned b) {
      mbar_arrive_expect_tx(&full[b % NS], bytes);
      bulk_g2s(smem + (b % NS) * bytes, base + (size_t)b * a.pitch, bytes, &full[b % NS], pol);
    };
    for (unsigned b = 0; b < nb && b < NS; ++b) load(b);
    for (unsigned b = 0; b < nb; ++b) {
      mbar_wait(&done[b % NS], (b / NS) & 1u);
      bulk_s2g(base + (size_t)b * a.pitch, smem + (b % NS) * bytes, bytes, pol);
      bulk_commit();
      if (b >= 1 && b - 1 + NS < nb) {
        bulk_wait_read<1>();
        load(b - 1 + NS);
      }
    }
    bulk_wait<0>();
    return;
  }
  // consumer warp: slot b is released when batch b + hold has landed
  for (unsigned b = 0; b < nb + a.hold; ++b) {
    if (b < nb) {
      mbar_wait(&full[b % NS], (b / NS) & 1u);
      if (a.touch) {
        float4* s = reinterpret_cast<float4*>(smem + (b % NS) * bytes);
        for (unsigned q = lane; q < a.piece / 4; q += 32) {
          float4 v = s[q];
          v.x *= 1.0000001f;
          s[q] = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
      }
    }
    if (b >= a.hold && lane == 0) mbar_arrive(&done[(b - a.hold) % NS]);
  }
}

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(t0);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(t1);
  CK(cudaEventSynchronize(t1));
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  return ms / reps;
}

template <int NS>
void run_bulk(float* P, size_t rows, unsigned cols, unsigned G, unsigned hold, int touch, int ef, int sms) {
  BulkArgs a;
  a.P = P;
  a.pitch = cols;
  a.G = G;
  a.piece = cols / G;
  const unsigned groups = sms / G;
  a.rows_per = rows / groups;
  a.hold = hold;
  a.touch = touch;
  a.evict_first = ef;
  const size_t smem = NS * (size_t)a.piece * 4 + 2 * NS * 8;
  CK(cudaFuncSetAttribute(rmw_bulk<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const double bytes = 2.0 * groups * a.rows_per * cols * 4;
  float ms = time_it([&] { rmw_bulk<NS><<<groups * G, 64, smem>>>(a); }, 10);
  CK(cudaGetLastError());
  printf("rmw_bulk NS=%2d slot=%6u B G=%u hold=%u touch=%d ef=%d : %.3f ms  %.0f GB/s\n", NS, a.piece * 4, G, hold,
         touch, ef, ms, bytes / ms / 1e6);
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n = (size_t)1 << 30;  // floats: 4 GiB
  float *P, *Q;
  CK(cudaMalloc(&P, n * 4));
  CK(cudaMalloc(&Q, n * 4));
  CK(cudaMemset(P, 0, n * 4));
  CK(cudaMemset(Q, 0, n * 4));
  const size_t n4 = n / 4;
  for (int blocks : {sms * 4, sms * 8, sms * 32}) {
    float ms = time_it([&] { copy_ldg<<<blocks, 512>>>((float4*)P, (float4*)Q, n4); }, 10);
    printf("copy_ldg   blocks=%5d : %.3f ms  %.0f GB/s\n", blocks, ms, 2.0 * n * 4 / ms / 1e6);
  }
  for (int blocks : {sms * 4, sms * 8}) {
    float ms = time_it([&] { rmw_ldg<1><<<blocks, 512>>>((float4*)P, n4); }, 10);
    printf("rmw_ldg<1> blocks=%5d : %.3f ms  %.0f GB/s\n", blocks, ms, 2.0 * n * 4 / ms / 1e6);
    ms = time_it([&] { rmw_ldg<4><<<blocks, 512>>>((float4*)P, n4); }, 10);
    printf("rmw_ldg<4> blocks=%5d : %.3f ms  %.0f GB/s\n", blocks, ms, 2.0 * n * 4 / ms / 1e6);
    ms = time_it([&] { rmw_ldg<8><<<blocks, 256>>>((float4*)P, n4); }, 10);
    printf("rmw_ldg<8> blocks=%5d : %.3f ms  %.0f GB/s\n", blocks, ms, 2.0 * n * 4 / ms / 1e6);
  }
  // 32768 x 32768, G = 4 pieces of 32 KiB (the headline layout)
  for (int ef : {1, 0}) {
    run_bulk<7>(P, 32768, 32768, 4, 0, 0, ef, sms);
    run_bulk<7>(P, 32768, 32768, 4, 3, 0, ef, sms);
  }
  run_bulk<7>(P, 32768, 32768, 4, 3, 1, 1, sms);
  run_bulk<6>(P, 32768, 32768, 4, 0, 0, 1, sms);
  run_bulk<4>(P, 32768, 32768, 4, 0, 0, 1, sms);
  // 16 KiB pieces (G = 8), 64 KiB pieces (G = 2)
  run_bulk<13>(P, 32768, 32768, 8, 0, 0, 1, sms);
  run_bulk<13>(P, 32768, 32768, 8, 3, 0, 1, sms);
  run_bulk<3>(P, 32768, 32768, 2, 0, 0, 1, sms);
  // contiguous 16 KiB rows (262144 x 4096, G = 1)
  run_bulk<13>(P, 262144, 4096, 1, 0, 0, 1, sms);
  run_bulk<13>(P, 262144, 4096, 1, 3, 0, 1, sms);
  run_bulk<7>(P, 131072, 8192, 1, 0, 0, 1, sms);
  return 0;
}
