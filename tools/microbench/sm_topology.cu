// Per-SM streaming speed vs GPU topology on B200 (scratch microbenchmark).
//
// Question: is the per-SM HBM bandwidth skew that makes a static row split
// slower than the dynamic batch counter a stable function of
// the SM's place in the chip (GPC / TPC), so that a STATIC split weighted by
// topology could be both deterministic and balanced?
//
//  A  dynamic TMA ring (producer warp, 32 KiB batches from a global counter),
//     per-SM batch counts averaged over reps, keyed by %smid;
//  B  static: every SM streams the same number of batches; per-SM elapsed
//     globaltimer ns under full concurrent load;
//  C  GPC membership from cluster launches: CTAs of one cluster share a GPC.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2412_11079_b200/csrc \
//      -o tools/microbench/sm_topology tools/microbench/sm_topology.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

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

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// DYN: batches from a global counter; else CTA c streams batches c, c+grid, ...
// (nper of them). Records smid, batches taken and elapsed ns per CTA.
template <int NS, bool DYN>
__global__ void __launch_bounds__(64, 1) ring(float* P, unsigned nbatch, unsigned bytes, unsigned* counter,
                                              unsigned* out_smid, unsigned* out_cnt, unsigned long long* out_ns) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * bytes);
  uint64_t* done = full + NS;
  unsigned* idx = reinterpret_cast<unsigned*>(done + NS);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&done[i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const unsigned long long t0 = gtimer();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = reinterpret_cast<unsigned char*>(P);
  unsigned seq = 0;
  if (warp == 0) {
    if (lane) return;
    const uint64_t pol = policy_evict_first();
    auto load = [&](unsigned b) {
      unsigned t;
      if (DYN) t = atomicAdd(counter, 1u);
      else t = blockIdx.x + seq++ * gridDim.x;
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
        out_cnt[blockIdx.x] = b;
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
    out_smid[blockIdx.x] = smid();
    out_ns[blockIdx.x] = gtimer() - t0;
    return;
  }
  for (unsigned b = 0;; ++b) {
    mbar_wait(&full[b % NS], (b / NS) & 1u);
    const unsigned t = idx[b % NS];
    if (lane == 0) mbar_arrive(&done[b % NS]);
    if (t >= nbatch) break;
  }
}

__global__ void cluster_probe(unsigned* out) {
  extern __shared__ unsigned char sm_[];
  if (threadIdx.x == 0) {
    sm_[0] = 1;
    unsigned cid;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
    out[2 * blockIdx.x] = smid();
    out[2 * blockIdx.x + 1] = cid;
  }
  // hold the SM so that the clusters of one launch are all resident together
  const unsigned long long t0 = gtimer();
  while (gtimer() - t0 < 200000) {
  }
}

struct UF {
  std::vector<int> p;
  explicit UF(int n) : p(n) { std::iota(p.begin(), p.end(), 0); }
  int f(int x) { return p[x] == x ? x : p[x] = f(p[x]); }
  void u(int a, int b) { p[f(a)] = f(b); }
};

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 5;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n = (size_t)1 << 30;  // 4 GiB of floats
  float* P;
  CK(cudaMalloc(&P, n * 4));
  fill_rand<<<sms * 8, 256>>>(P, n, 7);
  unsigned *counter, *d_smid, *d_cnt;
  unsigned long long* d_ns;
  CK(cudaMalloc(&counter, 4));
  CK(cudaMalloc(&d_smid, 4 * sms));
  CK(cudaMalloc(&d_cnt, 4 * sms));
  CK(cudaMalloc(&d_ns, 8 * sms));
  const unsigned bytes = 32768, nbatch = (unsigned)(n * 4 / bytes);
  const int smb = 7 * bytes + 256;
  CK(cudaFuncSetAttribute(ring<7, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));
  CK(cudaFuncSetAttribute(ring<7, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smb));
  std::vector<double> dyn(sms, 0.0), stat(sms, 0.0);
  std::vector<unsigned> h_smid(sms), h_cnt(sms);
  std::vector<unsigned long long> h_ns(sms);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < reps; ++r) {
    for (int d = 0; d < 2; ++d) {
      CK(cudaMemset(counter, 0, 4));
      cudaEventRecord(e0);
      if (d) ring<7, true><<<sms, 64, smb>>>(P, nbatch, bytes, counter, d_smid, d_cnt, d_ns);
      else ring<7, false><<<sms, 64, smb>>>(P, nbatch / sms * sms, bytes, counter, d_smid, d_cnt, d_ns);
      cudaEventRecord(e1);
      CK(cudaDeviceSynchronize());
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(h_smid.data(), d_smid, 4 * sms, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h_cnt.data(), d_cnt, 4 * sms, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h_ns.data(), d_ns, 8 * sms, cudaMemcpyDeviceToHost));
      const double gbs = 2.0 * (d ? nbatch : nbatch / sms * sms) * (double)bytes / (ms * 1e-3) / 1e9;
      printf("rep %d %s: %.3f ms %.0f GB/s\n", r, d ? "dyn" : "static", ms, gbs);
      for (int c = 0; c < sms; ++c) {
        if (d) dyn[h_smid[c]] += h_cnt[c];
        else stat[h_smid[c]] += h_ns[c] * 1e-6;
      }
    }
  }
  // GPC membership: clusters of C CTAs (one per SM) share a GPC
  UF uf(sms);
  CK(cudaFuncSetAttribute(cluster_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(cluster_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
  unsigned* d_out;
  CK(cudaMalloc(&d_out, 8 * 4 * sms));
  for (int C : {16, 8, 4, 2}) {
    for (int trial = 0; trial < 8; ++trial) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.blockDim = dim3(32);
      cfg.dynamicSmemBytes = 200000;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclus = 0;
      cfg.gridDim = dim3(C * 64);
      if (cudaOccupancyMaxActiveClusters(&nclus, cluster_probe, &cfg) != cudaSuccess || nclus < 1) {
        cudaGetLastError();
        printf("cluster %d: not launchable\n", C);
        break;
      }
      cfg.gridDim = dim3(C * nclus);
      if (cudaLaunchKernelEx(&cfg, cluster_probe, d_out) != cudaSuccess) {
        cudaGetLastError();
        printf("cluster %d: launch failed\n", C);
        break;
      }
      CK(cudaDeviceSynchronize());
      std::vector<unsigned> h(2 * C * nclus);
      CK(cudaMemcpy(h.data(), d_out, 8 * C * nclus, cudaMemcpyDeviceToHost));
      for (int b = 0; b < C * nclus; ++b)
        for (int b2 = b + 1; b2 < C * nclus; ++b2)
          if (h[2 * b + 1] == h[2 * b2 + 1] && h[2 * b] < (unsigned)sms && h[2 * b2] < (unsigned)sms)
            uf.u(h[2 * b], h[2 * b2]);
      if (trial == 0) printf("cluster %d: %d clusters resident (%d SMs)\n", C, nclus, C * nclus);
    }
  }
  std::vector<int> comp_size(sms, 0);
  for (int s = 0; s < sms; ++s) comp_size[uf.f(s)]++;
  printf("\nsmid gpc(root) gpc_size dyn_batches_avg static_ms_avg\n");
  for (int s = 0; s < sms; ++s)
    printf("%3d %3d %2d %8.1f %8.3f\n", s, uf.f(s), comp_size[uf.f(s)], dyn[s] / reps, stat[s] / reps);
  return 0;
}
