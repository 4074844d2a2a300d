// In-place RMW streaming mechanisms on B200 over random data (scratch microbenchmark).
//
// Which way of moving P through the SM reaches the HBM roofline for an
// in-place sweep, when the data are random (HBM power is data dependent):
//   tile_v4     torch-style: one short-lived CTA per contiguous tile, every
//               16-byte load of the thread issued up front, then the stores
//   tile_v8     the same with 32-byte (v8) global accesses
//   rows_reg    persistent CTA per SM streaming row slices (V float4 per thread
//               per row), D slices of prefetch held in registers
//   rows_cpa    persistent CTA per SM, per-thread cp.async (LDGSTS) into a
//               private smem ring of NS slices, LDS -> scale -> STG
//   rows_bulk   the product's mechanism: producer warp + cp.async.bulk ring
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
    p[i] = 0.5f + (x >> 8) * (1.0f / 16777216.0f);  // [0.5, 1.5): random mantissa bits
  }
}

constexpr float kC = 1.0000001f;

template <int TPB, int PER>
__global__ void __launch_bounds__(TPB) tile_v4(float4* a) {
  float4* t = a + (size_t)blockIdx.x * TPB * PER + threadIdx.x;
  float4 v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) v[k] = t[k * TPB];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    v[k].x *= kC; v[k].y *= kC; v[k].z *= kC; v[k].w *= kC;
    t[k * TPB] = v[k];
  }
}

struct f8 { float v[8]; };
__device__ __forceinline__ f8 ld8(const float* p) {
  f8 r;
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                 "=f"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st8(float* p, const f8& r) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]),
               "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
               : "memory");
}

template <int TPB, int PER>
__global__ void __launch_bounds__(TPB) tile_v8(float* a) {
  float* t = a + ((size_t)blockIdx.x * TPB * PER + threadIdx.x) * 8;
  f8 v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) v[k] = ld8(t + (size_t)k * TPB * 8);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[k].v[e] *= kC;
    st8(t + (size_t)k * TPB * 8, v[k]);
  }
}

// Persistent version of tile_v4: CTA b takes tiles b, b+grid, ... (static) or
// grabs the next tile from a global counter (dyn).
template <int TPB, int PER, bool DYN>
__global__ void __launch_bounds__(TPB) ptile_v4(float4* a, unsigned ntiles, unsigned* counter) {
  __shared__ unsigned next;
  unsigned tile = blockIdx.x;
  if (DYN) {
    if (threadIdx.x == 0) next = atomicAdd(counter, 1u);
    __syncthreads();
    tile = next;
  }
  while (tile < ntiles) {
    float4* t = a + (size_t)tile * TPB * PER + threadIdx.x;
    float4 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = t[k * TPB];
    if (DYN) {
      __syncthreads();
      if (threadIdx.x == 0) next = atomicAdd(counter, 1u);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      v[k].x *= kC; v[k].y *= kC; v[k].z *= kC; v[k].w *= kC;
      t[k * TPB] = v[k];
    }
    if (DYN) {
      __syncthreads();
      tile = next;
    } else {
      tile += gridDim.x;
    }
  }
}

// TMA ring over contiguous rows (G = 1) whose producer grabs the next batch of
// R rows from a global counter: all SMs stream one moving window of the matrix.
template <int NS>
__global__ void __launch_bounds__(64, 1) rows_bulk_dyn(float* P, unsigned nbatch, unsigned bytes, unsigned* counter,
                                                     unsigned* per_cta) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * bytes);
  uint64_t* done = full + NS;
  unsigned* idx = reinterpret_cast<unsigned*>(done + NS);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&done[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = reinterpret_cast<unsigned char*>(P);
  if (warp == 0) {
    if (lane) return;
    const uint64_t pol = policy_evict_first();
    auto load = [&](unsigned b) {  // slot b: grab a batch, or post an empty sentinel
      const unsigned t = atomicAdd(counter, 1u);
      idx[b % NS] = t;
      if (t < nbatch) {
        mbar_arrive_expect_tx(&full[b % NS], bytes);
        bulk_g2s(smem + (b % NS) * bytes, base + (size_t)t * bytes, bytes, &full[b % NS], pol);
      } else {
        mbar_arrive(&full[b % NS]);
      }
    };
    for (unsigned b = 0; b < NS; ++b) load(b);
    for (unsigned b = 0;; ++b) {
      mbar_wait(&done[b % NS], (b / NS) & 1u);
      const unsigned t = idx[b % NS];
      if (t >= nbatch) {
        per_cta[blockIdx.x] = b;
        break;
      }
      bulk_s2g(base + (size_t)t * bytes, smem + (b % NS) * bytes, bytes, pol);
      bulk_commit();
      if (b >= 1) {
        bulk_wait_read<1>();
        load(b - 1 + NS);
      }
    }
    bulk_wait<0>();
    return;
  }
  for (unsigned b = 0;; ++b) {
    mbar_wait(&full[b % NS], (b / NS) & 1u);
    const unsigned t = idx[b % NS];
    if (lane == 0) mbar_arrive(&done[b % NS]);
    if (t >= nbatch) break;
  }
}

// [rows][pitch] matrix, G CTAs per row (slice = pitch/G floats = 4*NT*V),
// group c/G takes rows interleaved (il) or a contiguous block.
struct RowArgs {
  float* P;
  unsigned rows, pitch, G, groups;
  int il;
};
__device__ __forceinline__ size_t row_index(const RowArgs& a, unsigned grp, unsigned s) {
  return a.il ? (size_t)s * a.groups + grp : (size_t)grp * (a.rows / a.groups) + s;
}

template <int NT, int V, int D>
__global__ void __launch_bounds__(NT, 1) rows_reg(const RowArgs a) {
  const unsigned grp = blockIdx.x / a.G, g = blockIdx.x % a.G;
  const unsigned nb = a.rows / a.groups;
  const unsigned slice = a.pitch / a.G;
  auto ptr = [&](unsigned s) {
    return reinterpret_cast<float4*>(a.P + row_index(a, grp, s) * a.pitch + (size_t)g * slice) + threadIdx.x;
  };
  float4 buf[D][V];
#pragma unroll
  for (int d = 0; d < D; ++d)
    if (d < (int)nb)
#pragma unroll
      for (int k = 0; k < V; ++k) buf[d][k] = ptr(d)[k * NT];
  for (unsigned s0 = 0; s0 < nb; s0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const unsigned s = s0 + d;
      if (s < nb) {
        float4 v[V];
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = buf[d][k];
        if (s + D < nb)
#pragma unroll
          for (int k = 0; k < V; ++k) buf[d][k] = ptr(s + D)[k * NT];
        float4* p = ptr(s);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          v[k].x *= kC; v[k].y *= kC; v[k].z *= kC; v[k].w *= kC;
          p[k * NT] = v[k];
        }
      }
    }
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NT, int V, int NS>
__global__ void __launch_bounds__(NT, 1) rows_cpa(const RowArgs a) {
  extern __shared__ __align__(128) float4 ring[];  // [NS][V][NT]
  const unsigned grp = blockIdx.x / a.G, g = blockIdx.x % a.G;
  const unsigned nb = a.rows / a.groups;
  const unsigned slice = a.pitch / a.G;
  auto ptr = [&](unsigned s) {
    return reinterpret_cast<float4*>(a.P + row_index(a, grp, s) * a.pitch + (size_t)g * slice) + threadIdx.x;
  };
  auto issue = [&](unsigned s) {
    if (s < nb) {
      const float4* p = ptr(s);
#pragma unroll
      for (int k = 0; k < V; ++k) cp_async16(&ring[((s % NS) * V + k) * NT + threadIdx.x], p + k * NT);
    }
    cp_commit();
  };
#pragma unroll
  for (int d = 0; d < NS - 1; ++d) issue(d);
  for (unsigned s = 0; s < nb; ++s) {
    issue(s + NS - 1);
    cp_wait<NS - 1>();
    float4* p = ptr(s);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      float4 v = ring[((s % NS) * V + k) * NT + threadIdx.x];
      v.x *= kC; v.y *= kC; v.z *= kC; v.w *= kC;
      p[k * NT] = v;
    }
  }
}

template <int NS>
__global__ void __launch_bounds__(64, 1) rows_bulk(const RowArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned slice = a.pitch / a.G;
  const unsigned bytes = slice * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * bytes);
  uint64_t* done = full + NS;
  const unsigned grp = blockIdx.x / a.G, g = blockIdx.x % a.G;
  const unsigned nb = a.rows / a.groups;
  auto gptr = [&](unsigned s) { return a.P + row_index(a, grp, s) * a.pitch + (size_t)g * slice; };
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&done[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane) return;
    const uint64_t pol = policy_evict_first();
    auto load = [&](unsigned b) {
      mbar_arrive_expect_tx(&full[b % NS], bytes);
      bulk_g2s(smem + (b % NS) * bytes, gptr(b), bytes, &full[b % NS], pol);
    };
    for (unsigned b = 0; b < nb && b < NS; ++b) load(b);
    for (unsigned b = 0; b < nb; ++b) {
      mbar_wait(&done[b % NS], (b / NS) & 1u);
      bulk_s2g(gptr(b), smem + (b % NS) * bytes, bytes, pol);
      bulk_commit();
      if (b >= 1 && b - 1 + NS < nb) {
        bulk_wait_read<1>();
        load(b - 1 + NS);
      }
    }
    bulk_wait<0>();
    return;
  }
  for (unsigned b = 0; b < nb; ++b) {
    mbar_wait(&full[b % NS], (b / NS) & 1u);
    if (lane == 0) mbar_arrive(&done[b % NS]);
  }
}

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

int main(int argc, char** argv) {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int reps = argc > 1 ? atoi(argv[1]) : 10;
  const char* only = argc > 2 ? argv[2] : "";
  const size_t n = (size_t)1 << 30;  // 4 GiB of floats
  float* P;
  CK(cudaMalloc(&P, n * 4));
  fill_rand<<<sms * 8, 512>>>(P, n, 12345u);
  CK(cudaDeviceSynchronize());
  auto want = [&](const char* name) { return !*only || strstr(name, only); };
  auto report = [&](const char* name, double bytes, float ms) {
    printf("%-34s %.3f ms  %5.0f GB/s\n", name, ms, bytes / ms / 1e6);
    fflush(stdout);
  };
  const double all = 2.0 * n * 4;
  if (want("tile_v4")) {
    report("tile_v4<256,4>", all, time_it([&] { tile_v4<256, 4><<<n / 4 / 1024, 256>>>((float4*)P); }, reps));
    report("tile_v4<128,8>", all, time_it([&] { tile_v4<128, 8><<<n / 4 / 1024, 128>>>((float4*)P); }, reps));
    report("tile_v4<256,8>", all, time_it([&] { tile_v4<256, 8><<<n / 4 / 2048, 256>>>((float4*)P); }, reps));
  }
  if (want("tile_v8")) {
    report("tile_v8<256,2>", all, time_it([&] { tile_v8<256, 2><<<n / 8 / 512, 256>>>(P); }, reps));
    report("tile_v8<256,4>", all, time_it([&] { tile_v8<256, 4><<<n / 8 / 1024, 256>>>(P); }, reps));
    report("tile_v8<128,4>", all, time_it([&] { tile_v8<128, 4><<<n / 8 / 512, 128>>>(P); }, reps));
  }
  unsigned *counter, *per_cta;
  CK(cudaMalloc(&counter, 4));
  CK(cudaMalloc(&per_cta, 4096));
  if (want("ptile")) {
    const unsigned nt = n / 4 / 1024;
    for (int cps : {4, 8}) {
      char name[64];
      snprintf(name, sizeof name, "ptile_v4<256,4> static cps=%d", cps);
      report(name, all, time_it([&] { ptile_v4<256, 4, false><<<sms * cps, 256>>>((float4*)P, nt, counter); }, reps));
      snprintf(name, sizeof name, "ptile_v4<256,4> dyn cps=%d", cps);
      report(name, all, time_it([&] {
        cudaMemsetAsync(counter, 0, 4);
        ptile_v4<256, 4, true><<<sms * cps, 256>>>((float4*)P, nt, counter);
      }, reps));
    }
  }
  if (want("bulk_dyn")) {
    for (unsigned bytes : {16384u, 32768u}) {
      const unsigned nbatch = (unsigned)(n * 4 / bytes);
      const int smb = 7 * bytes + 256;
      CK(cudaFuncSetAttribute(rows_bulk_dyn<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));
      char name[64];
      snprintf(name, sizeof name, "rows_bulk_dyn<7> batch=%u B", bytes);
      report(name, all, time_it([&] {
        cudaMemsetAsync(counter, 0, 4);
        rows_bulk_dyn<7><<<sms, 64, smb>>>(P, nbatch, bytes, counter, per_cta);
      }, reps));
      unsigned h[1024];
      CK(cudaMemcpy(h, per_cta, sms * 4, cudaMemcpyDeviceToHost));
      unsigned mn = ~0u, mx = 0;
      double sum = 0;
      for (int c = 0; c < sms; ++c) { mn = h[c] < mn ? h[c] : mn; mx = h[c] > mx ? h[c] : mx; sum += h[c]; }
      int smid_of[1024];
      (void)smid_of;
      printf("  batches per CTA: min %u max %u mean %.1f\n  ", mn, mx, sum / sms);
      for (int c = 0; c < sms; ++c) printf("%u%s", h[c], c % 37 == 36 ? "\n  " : " ");
      printf("\n");
    }
  }
  // row-slice shapes: 32768 x 32768 (G=4, slice 8192) and 262144 x 4096 (G=1)
  struct Shape { unsigned rows, cols, G; };
  for (Shape sh : {Shape{32768, 32768, 4}, Shape{262144, 4096, 1}}) {
    for (int il = 0; il < 2; ++il) {
      RowArgs a;
      a.P = P;
      a.pitch = sh.cols;
      a.G = sh.G;
      a.groups = sms / sh.G;
      a.rows = sh.rows / a.groups * a.groups;
      a.il = il;
      const double bytes = 2.0 * a.rows * a.pitch * 4;
      char name[96];
      const unsigned slice = sh.cols / sh.G;
      if (slice == 8192) {
        if (want("rows_reg")) {
          snprintf(name, sizeof name, "rows_reg<512,4,2> %ux%u il=%d", a.rows, a.pitch, il);
          report(name, bytes, time_it([&] { rows_reg<512, 4, 2><<<a.groups * a.G, 512>>>(a); }, reps));
          snprintf(name, sizeof name, "rows_reg<1024,2,4> %ux%u il=%d", a.rows, a.pitch, il);
          report(name, bytes, time_it([&] { rows_reg<1024, 2, 4><<<a.groups * a.G, 1024>>>(a); }, reps));
        }
        if (want("rows_cpa")) {
          const int sm4 = 4 * 4 * 512 * 16;
          CK(cudaFuncSetAttribute(rows_cpa<512, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
          snprintf(name, sizeof name, "rows_cpa<512,4,4> %ux%u il=%d", a.rows, a.pitch, il);
          report(name, bytes, time_it([&] { rows_cpa<512, 4, 4><<<a.groups * a.G, 512, sm4>>>(a); }, reps));
          const int sm6 = 6 * 4 * 512 * 16;
          CK(cudaFuncSetAttribute(rows_cpa<512, 4, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm6));
          snprintf(name, sizeof name, "rows_cpa<512,4,6> %ux%u il=%d", a.rows, a.pitch, il);
          report(name, bytes, time_it([&] { rows_cpa<512, 4, 6><<<a.groups * a.G, 512, sm6>>>(a); }, reps));
        }
      } else {
        if (want("rows_reg")) {
          snprintf(name, sizeof name, "rows_reg<512,2,4> %ux%u il=%d", a.rows, a.pitch, il);
          report(name, bytes, time_it([&] { rows_reg<512, 2, 4><<<a.groups * a.G, 512>>>(a); }, reps));
          snprintf(name, sizeof name, "rows_reg<1024,1,6> %ux%u il=%d", a.rows, a.pitch, il);
          report(name, bytes, time_it([&] { rows_reg<1024, 1, 6><<<a.groups * a.G, 1024>>>(a); }, reps));
        }
        if (want("rows_cpa")) {
          const int sm8 = 8 * 2 * 512 * 16;
          CK(cudaFuncSetAttribute(rows_cpa<512, 2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8));
          snprintf(name, sizeof name, "rows_cpa<512,2,8> %ux%u il=%d", a.rows, a.pitch, il);
          report(name, bytes, time_it([&] { rows_cpa<512, 2, 8><<<a.groups * a.G, 512, sm8>>>(a); }, reps));
          const int sm12 = 12 * 2 * 512 * 16;
          CK(cudaFuncSetAttribute(rows_cpa<512, 2, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm12));
          snprintf(name, sizeof name, "rows_cpa<512,2,12> %ux%u il=%d", a.rows, a.pitch, il);
          report(name, bytes, time_it([&] { rows_cpa<512, 2, 12><<<a.groups * a.G, 512, sm12>>>(a); }, reps));
        }
      }
      if (want("rows_bulk")) {
        const int smb = 7 * slice * 4 + 256;
        CK(cudaFuncSetAttribute(rows_bulk<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));
        snprintf(name, sizeof name, "rows_bulk<7> %ux%u il=%d", a.rows, a.pitch, il);
        report(name, bytes, time_it([&] { rows_bulk<7><<<a.groups * a.G, 64, smb>>>(a); }, reps));
      }
    }
  }
  CK(cudaFree(P));
  return 0;
}
