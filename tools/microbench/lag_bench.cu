// Pipeline mechanics for the fused sweep's alpha lag (scratch microbenchmark).
//
// The product kernel holds each row batch in its shared-memory ring slot from
// the TMA load until sweep 2 (LA + 2 batches later) and the bulk store: of its
// 7 x 32 KiB slots only ~2 carry loads in flight. This measures in-place RMW
// streaming of 4 GiB of random floats in 32 KiB batches with
//   bulk      TMA load -> consumers -> TMA bulk store from the same slot (rows_bulk_dyn)
//   stg L     TMA load -> LDS -> (L > 0: park the batch in the thread's TMEM lane
//             for L batches, tcgen05.st / tcgen05.ld) -> STG from registers;
//             the smem slot is free right after the LDS, so every slot loads.
//   hold L    TMA load -> LDS -> slot held L more batches -> STS -> TMA bulk store
//             (the product's mechanism without the arithmetic)
// with batches from a global counter (dyn) or static contiguous blocks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2412_11079_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace uotk;

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void fill_rand(float* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 15; x *= 2246822519u; x ^= x >> 13; x *= 3266489917u; x ^= x >> 16;
    p[i] = 0.5f + (x >> 8) * (1.0f / 16777216.0f);
  }
}

constexpr float kC = 1.0000001f;
constexpr unsigned kBytes = 32768;           // one batch = one 8192-float row slice
constexpr int NT = 512, NW = NT / 32, V = 4;  // 16 floats per compute thread

__device__ __forceinline__ void tm_st16(uint32_t taddr, const float4 (&v)[V]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "f"(v[0].x), "f"(v[0].y), "f"(v[0].z), "f"(v[0].w), "f"(v[1].x), "f"(v[1].y), "f"(v[1].z), "f"(v[1].w),
      "f"(v[2].x), "f"(v[2].y), "f"(v[2].z), "f"(v[2].w), "f"(v[3].x), "f"(v[3].y), "f"(v[3].z), "f"(v[3].w)
      : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, float4 (&v)[V]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[0].z), "=f"(v[0].w), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[1].z),
        "=f"(v[1].w), "=f"(v[2].x), "=f"(v[2].y), "=f"(v[2].z), "=f"(v[2].w), "=f"(v[3].x), "=f"(v[3].y),
        "=f"(v[3].z), "=f"(v[3].w)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// MODE 0: stg (LAG batches parked in TMEM, 0 = none); MODE 1: hold (slot held LAG batches, bulk store)
template <int NS, int LAG, int MODE, bool DYN>
__global__ void __launch_bounds__(NT + 32, 1) lag_kernel(float* P, unsigned nbatch, unsigned* counter, unsigned* per_cta) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * kBytes);
  uint64_t* freeb = full + NS;
  unsigned* idx = reinterpret_cast<unsigned*>(freeb + NS);
  uint32_t* tm = idx + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&freeb[i], NW); }
    fence_mbar_init();
  }
  constexpr bool TM = MODE == 0 && LAG > 0;
  if (TM && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tm)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = TM ? *tm : 0u;
  const unsigned per = (nbatch + gridDim.x - 1) / gridDim.x;
  const unsigned b0 = blockIdx.x * per, b1 = min(nbatch, b0 + per);
  unsigned char* base = reinterpret_cast<unsigned char*>(P);

  if (warp == NW) {
    if (lane) return;
    const uint64_t pol = policy_evict_first();
    auto load = [&](unsigned b) {
      unsigned t;
      if (DYN) t = atomicAdd(counter, 1u);
      else t = b0 + b < b1 ? b0 + b : ~0u;
      if (t >= nbatch) t = ~0u;
      idx[b % NS] = t;
      if (t != ~0u) {
        mbar_arrive_expect_tx(&full[b % NS], kBytes);
        bulk_g2s(smem + (b % NS) * kBytes, base + (size_t)t * kBytes, kBytes, &full[b % NS], pol);
      } else {
        mbar_arrive(&full[b % NS]);
      }
    };
    for (unsigned b = 0; b < NS; ++b) load(b);
    for (unsigned b = 0;; ++b) {
      mbar_wait(&freeb[b % NS], (b / NS) & 1u);
      const unsigned t = idx[b % NS];
      if (t == ~0u) { per_cta[blockIdx.x] = b; break; }
      if (MODE == 1) {
        bulk_s2g(base + (size_t)t * kBytes, smem + (b % NS) * kBytes, kBytes, pol);
        bulk_commit();
        bulk_wait_read<0>();
      }
      load(b + NS);
    }
    if (MODE == 1) bulk_wait<0>();
    return;
  }
  // compute warps
  const uint32_t tcol = tbase + (static_cast<uint32_t>(32 * (warp % 4)) << 16) + 16 * (warp / 4);
  unsigned tq[LAG + 1];
#pragma unroll
  for (int i = 0; i <= LAG; ++i) tq[i] = ~0u;
  unsigned nb = ~0u;
  for (unsigned s = 0;; ++s) {
    float4 v[V];
    bool have = false;
    if (s < nb) {
      mbar_wait(&full[s % NS], (s / NS) & 1u);
      const unsigned t = idx[s % NS];
      if (t == ~0u) {
        nb = s;
        if (MODE == 0 || LAG == 0) { __syncwarp(); if (lane == 0) mbar_arrive(&freeb[s % NS]); }
      } else {
        have = true;
        const float4* src = reinterpret_cast<const float4*>(smem + (s % NS) * kBytes);
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = src[tid + k * NT];
#pragma unroll
        for (int k = 0; k < V; ++k) { v[k].x *= kC; v[k].y *= kC; v[k].z *= kC; v[k].w *= kC; }
        if (MODE == 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&freeb[s % NS]);  // slot free right after the reads
          if (LAG == 0) {
            float4* dst = reinterpret_cast<float4*>(base + (size_t)t * kBytes);
#pragma unroll
            for (int k = 0; k < V; ++k) __stcs(&dst[tid + k * NT], v[k]);
          } else {
            tm_st16(tcol + 64 * (s % (LAG + 1)), v);
          }
        }
        tq[s % (LAG + 1)] = t;
      }
    }
    if (LAG > 0 && s >= static_cast<unsigned>(LAG) && s - LAG < nb) {
      const unsigned b = s - LAG;
      if (MODE == 0) {
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        float4 w[V];
        tm_ld16(tcol + 64 * (b % (LAG + 1)), w);
        float4* dst = reinterpret_cast<float4*>(base + (size_t)tq[b % (LAG + 1)] * kBytes);
#pragma unroll
        for (int k = 0; k < V; ++k) __stcs(&dst[tid + k * NT], w[k]);
      } else {
        float4* buf = reinterpret_cast<float4*>(smem + (b % NS) * kBytes);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          float4 w = buf[tid + k * NT];
          w.x *= kC; w.y *= kC; w.z *= kC; w.w *= kC;
          buf[tid + k * NT] = w;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&freeb[b % NS]);
      }
    }
    if (MODE == 1 && LAG == 0 && have) {
      float4* buf = reinterpret_cast<float4*>(smem + (s % NS) * kBytes);
#pragma unroll
      for (int k = 0; k < V; ++k) buf[tid + k * NT] = v[k];
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&freeb[s % NS]);
    }
    if (!have && s >= nb + LAG) {
      if (MODE == 1 && LAG > 0) {  // the sentinel slot: release it so the producer sees it
        __syncwarp();
        if (lane == 0) mbar_arrive(&freeb[nb % NS]);
      }
      break;
    }
  }
  if (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
    }
  }
}

template <class F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  CK(cudaGetLastError());
  return best;
}

int main(int argc, char** argv) {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int reps = argc > 1 ? atoi(argv[1]) : 10;
  const size_t n = (size_t)1 << 30;
  float* P;
  CK(cudaMalloc(&P, n * 4));
  fill_rand<<<sms * 8, 512>>>(P, n, 12345u);
  unsigned *counter, *per_cta;
  CK(cudaMalloc(&counter, 4));
  CK(cudaMalloc(&per_cta, 4096));
  CK(cudaDeviceSynchronize());
  const unsigned nbatch = (unsigned)(n * 4 / kBytes);
  const double all = 2.0 * n * 4;
  auto run = [&](const char* name, auto kern, int ns) {
    const int smb = ns * kBytes + 256;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));
    float ms = time_it([&] {
      cudaMemsetAsync(counter, 0, 4);
      kern<<<sms, NT + 32, smb>>>(P, nbatch, counter, per_cta);
    }, reps);
    printf("%-28s %.3f ms  %5.0f GB/s\n", name, ms, all / ms / 1e6);
    fflush(stdout);
  };
  run("hold L=0 dyn  (bulk)", lag_kernel<7, 0, 1, true>, 7);
  run("hold L=3 dyn  (product)", lag_kernel<7, 3, 1, true>, 7);
  run("hold L=3 static", lag_kernel<7, 3, 1, false>, 7);
  run("stg L=0 dyn", lag_kernel<7, 0, 0, true>, 7);
  run("stg L=0 static", lag_kernel<7, 0, 0, false>, 7);
  run("stg L=3 dyn  (TMEM lag)", lag_kernel<7, 3, 0, true>, 7);
  run("stg L=3 static", lag_kernel<7, 3, 0, false>, 7);
  run("stg L=5 dyn", lag_kernel<7, 5, 0, true>, 7);
  run("stg L=5 static", lag_kernel<7, 5, 0, false>, 7);
  run("stg L=3 dyn ns=6", lag_kernel<6, 3, 0, true>, 6);
  run("hold L=3 dyn ns=6", lag_kernel<6, 3, 1, true>, 6);
  return 0;
}
