// Flag block of a rank's symmetric allocation (dist.py FLAG_BYTES) shared by every kernel
// that writes into peers' receive regions: the a2a push kernels (a2a.cu) and the fused
// attention-forward + head->seq push (attn_fwd.cu).  Words are uint32.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace autosp {

constexpr int kReadyWord = 0;     // "this rank reached epoch e" (its older readers are done)
constexpr int kArriveWord = 16;   // + src rank: src finished writing call e into me
constexpr int kCheckWord = 32;    // + src rank: sender's view of the destination offset
constexpr int kCounterWord = 48;  // 8 CTA completion counters (local use only), one per
constexpr int kCounterSlots = 8;  // epoch mod 8: consecutive calls never share a counter

// Completion of a launch that pushed into peers: every thread's (remote) stores are
// ordered before thread 0's system-scope fence by the CTA barrier (fences are
// cumulative); the last CTA to finish publishes arrive[rank] = epoch (+ check word) in
// every peer's flag block.  Must be called by all threads of every CTA.
// AUTOSP_GPU_FENCE_CTAS=1: every CTA fences at gpu scope and only the last one at system
// scope (cumulativity through the gpu-scope counter atomics): -13 % per small loopback
// call, but it leans on cross-scope cumulativity for NVLink peer writes that one GPU cannot
// test, so the default keeps a system-scope fence per CTA.
#ifndef AUTOSP_GPU_FENCE_CTAS
#define AUTOSP_GPU_FENCE_CTAS 0
#endif
AUTOSP_DEV void publish_arrival(uint32_t* const* peer_flags, int P, int rank, uint32_t epoch,
                                uint32_t check, uint32_t n_ctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (AUTOSP_GPU_FENCE_CTAS) __threadfence();
    else __threadfence_system();
    uint32_t* ctr = peer_flags[rank] + kCounterWord + (epoch % kCounterSlots);
    const uint32_t old = atom_add_acqrel_gpu(ctr, 1u);
    if (old == n_ctas - 1) {
      *ctr = 0u;
      __threadfence_system();
      for (int j = 0; j < P; ++j)
        if (j != rank) {
          peer_flags[j][kCheckWord + rank] = check;
          st_release_sys(peer_flags[j] + kArriveWord + rank, epoch);
        }
    }
  }
}

// Check word of one call: FNV-1a over every destination descriptor (offset, strides,
// heads) of the call, computed by the sender from its descriptors and by the receiver from
// its own; a2a_wait traps when they differ (the symmetric-allocation invariant).
struct CheckHash {
  uint32_t h = 2166136261u;
  void add(int64_t v) {
    uint64_t u = static_cast<uint64_t>(v);
    for (int i = 0; i < 8; ++i) {
      h ^= static_cast<uint32_t>(u & 0xffu);
      h *= 16777619u;
      u >>= 8;
    }
  }
};

}  // namespace autosp
