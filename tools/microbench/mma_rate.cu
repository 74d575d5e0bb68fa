// Measure tcgen05.mma issue->completion throughput for SS and TS variants at several N
// (development microbenchmark; not part of the library).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_27089_b200/csrc/ptx.cuh"
using namespace autosp;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tm);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tm;
  const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, 0, TS ? 1 : 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      if (TS)
        mma_ts(t + 256, t + kk * 8, make_smem_desc(sb + kk * 2048, 16384, 1024, 2), idesc, 1);
      else
        mma_ss(t + 256, make_smem_desc(sa + kk * 32, 16, 1024, 2),
               make_smem_desc(sb + kk * 32, 16, 1024, 2), idesc, 1);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

template <int N, bool TS>
void run(int blocks) {
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  auto k = mma_rate<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  const int iters = 4096;
  k<<<blocks, 128, 100000>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double flops = 2.0 * 128 * N * 16;
  printf("%s N=%3d blocks=%3d: %.1f cycles/mma  (%.0f flop/cycle/SM; floor %d)  err=%s\n",
         TS ? "TS" : "SS", N, blocks, avg / iters, flops * iters / avg, 128 * N / 256,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int b : {1, 148}) {
    run<64, false>(b); run<128, false>(b); run<256, false>(b);
    run<64, true>(b); run<128, true>(b); run<256, true>(b);
  }
}
