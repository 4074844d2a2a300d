// topology.cuh — per-SM HBM streaming speed classes of the GPU (B200).
//
// Measured on B200 (tools/microbench/sm_topology.cu, profiles/r02_topology.md):
// when every SM streams the same bytes in place through a cp.async.bulk ring,
// the per-SM elapsed times fall into a few crisp classes (0.82 / 1.18 / 1.33 ms,
// +-1%), constant per TPC (SM pair 2k, 2k+1) and stable run to run. A static
// equal row split is paced by the slowest class; the dynamic batch counter
// balances it but makes the f64 column sums run dependent. The sweep's
// deterministic schedule therefore (1) groups the CTAs of a row group on SMs of
// ONE class and (2) gives every row group a row count proportional to its
// class's speed — a static split, bit-reproducible on a given GPU.
//
// sm_probe_kernel: one CTA per SM (cooperative, forced by its shared-memory
// footprint); a producer thread streams `nb` batches of 32 KiB through a
// 6-slot ring (bulk load -> bulk store back, in place) over its own region of
// a scratch buffer and records the elapsed globaltimer ns under its %smid.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace uotk {

constexpr int kProbeSlots = 6;
constexpr unsigned kProbeBytes = 32768;

__global__ void __launch_bounds__(32, 1) sm_probe_kernel(unsigned char* buf, unsigned nb,
                                                        unsigned long long* out_ns) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kProbeSlots * kProbeBytes);
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kProbeSlots; ++i) mbar_init(&full[i], 1);
  fence_mbar_init();
  unsigned char* base = buf + static_cast<size_t>(blockIdx.x) * nb * kProbeBytes;
  const uint64_t pol = policy_evict_first();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (unsigned b = 0; b < kProbeSlots && b < nb; ++b) {
    mbar_arrive_expect_tx(&full[b], kProbeBytes);
    bulk_g2s(smem + b * kProbeBytes, base + static_cast<size_t>(b) * kProbeBytes, kProbeBytes, &full[b], pol);
  }
  for (unsigned b = 0; b < nb; ++b) {
    const unsigned s = b % kProbeSlots;
    mbar_wait(&full[s], (b / kProbeSlots) & 1u);
    bulk_s2g(base + static_cast<size_t>(b) * kProbeBytes, smem + s * kProbeBytes, kProbeBytes, pol);
    bulk_commit();
    // refill the slot of the previous batch once its store has read it
    if (b >= 1 && b - 1 + kProbeSlots < nb) {
      const unsigned r = (b - 1) % kProbeSlots;
      bulk_wait_read<1>();
      mbar_arrive_expect_tx(&full[r], kProbeBytes);
      bulk_g2s(smem + r * kProbeBytes, base + static_cast<size_t>(b - 1 + kProbeSlots) * kProbeBytes, kProbeBytes,
               &full[r], pol);
    }
  }
  bulk_wait<0>();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out_ns[smid()] = t1 - t0;
}

inline size_t sm_probe_smem() { return kProbeSlots * kProbeBytes + kProbeSlots * 8; }

}  // namespace uotk
