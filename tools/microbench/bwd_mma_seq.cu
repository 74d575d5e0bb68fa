// Pure tensor-pipe time of one attention-backward step (d = 64) with the EXACT operand
// descriptors of attn_bwd_kernel<64>: S^T (SS, K-major), dP^T (SS), dV (TS, B MN-major),
// dK (TS, B MN-major), dQ (SS, A = dS^T MN-major, B = K MN-major).  One thread issues
// `steps` steps back to back with no dependencies; prints cycles per step for the full
// sequence and for each group alone (development microbenchmark).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_27089_b200/csrc/ptx.cuh"
using namespace autosp;

constexpr int SW = 128, SBO = 1024, LAYOUT = 2, TILE = 128 * 64 * 2;

template <int MASK>  // bit0 S, bit1 dP, bit2 dV, bit3 dK, bit4 dQ
__global__ void __launch_bounds__(128, 1) seq(long long* out, int steps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tm);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tm;
  const uint32_t s_k = smem_u32(smem), s_v = s_k + TILE, s_q = s_v + TILE, s_do = s_q + TILE,
                 s_ds = s_do + TILE;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idesc_g = make_idesc_bf16(128, 64, 0, 1);
    constexpr uint32_t idesc_q = make_idesc_bf16(128, 64, 1, 1);
    const uint64_t dk_k = make_smem_desc(s_k, 16, SBO, LAYOUT), dv_k = make_smem_desc(s_v, 16, SBO, LAYOUT);
    const uint64_t dq_k = make_smem_desc(s_q, 16, SBO, LAYOUT), ddo_k = make_smem_desc(s_do, 16, SBO, LAYOUT);
    const uint64_t dq_mn = make_smem_desc(s_q, 128 * SW, SBO, LAYOUT), ddo_mn = make_smem_desc(s_do, 128 * SW, SBO, LAYOUT);
    const uint64_t dk_mn = make_smem_desc(s_k, 128 * SW, SBO, LAYOUT);
    const uint64_t dds = make_smem_desc(s_ds, 128 * 128, 1024, 2);
    auto pk = [](int kk) -> uint32_t { return kk < 4 ? kk * 8 : 96 + (kk - 4) * 8; };
    long long t0 = clock64();
    for (int st = 0; st < steps; ++st) {
      const uint32_t sc = (st & 1) * 128;
      if (MASK & 1)
        for (int kk = 0; kk < 4; ++kk) mma_ss(t + sc, dk_k + 2 * kk, dq_k + 2 * kk, idesc_s, kk > 0);
      if (MASK & 2)
        for (int kk = 0; kk < 4; ++kk) mma_ss(t + 256, dv_k + 2 * kk, ddo_k + 2 * kk, idesc_s, kk > 0);
      if (MASK & 4)
        for (int kk = 0; kk < 8; ++kk) mma_ts(t + 384, t + sc + pk(kk), ddo_mn + ((kk * 16 * SW) >> 4), idesc_g, 1);
      if (MASK & 8)
        for (int kk = 0; kk < 8; ++kk) mma_ts(t + 448, t + 256 + pk(kk), dq_mn + ((kk * 16 * SW) >> 4), idesc_g, 1);
      if (MASK & 16)
        for (int kk = 0; kk < 8; ++kk) mma_ss(t + sc + 32, dds + ((kk * 16 * 128) >> 4), dk_mn + ((kk * 16 * SW) >> 4), idesc_q, kk > 0);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

template <int MASK>
void run(const char* name, int blocks) {
  long long* d;
  cudaMalloc(&d, 256 * sizeof(long long));
  const int steps = 2000;
  auto k = seq<MASK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * TILE + 2048);
  k<<<blocks, 128, 6 * TILE + 2048>>>(d, 10);
  k<<<blocks, 128, 6 * TILE + 2048>>>(d, steps);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  printf("%-22s blocks=%3d: %7.1f cycles/step  err=%s\n", name, blocks, avg / steps,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int b : {1, 148}) {
    run<31>("full step", b);
    run<3>("S+dP (SS N128)", b);
    run<12>("dV+dK (TS N64)", b);
    run<16>("dQ (SS MN-major)", b);
    run<1>("S only", b);
    run<4>("dV only", b);
  }
}
