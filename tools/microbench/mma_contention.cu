// MMA throughput while other warps stream TMEM loads/stores (softmax-like traffic).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_27089_b200/csrc/ptx.cuh"
using namespace autosp;

template <int N, bool TS, int MODE>  // MODE 0: idle, 1: ld x32 loop, 2: ld+st loop, 3: FMA loop
__global__ void __launch_bounds__(384, 1) mma_cont(long long* out, int iters, int* stop) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tm);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); done = 0; }
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
    done = 1;
  } else if (warp >= 4) {
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t r[32];
    float acc = 0.f;
    long long n = 0;
    while (!done) {
      if (MODE == 1 || MODE == 2) {
        tmem_ld32(t + lane_base + (warp >= 8 ? 128 : 0), r);
        tmem_wait_ld();
        if (MODE == 2) {
          tmem_st32(t + lane_base + (warp >= 8 ? 128 : 0) + 64, r);
          tmem_wait_st();
        }
        acc += __uint_as_float(r[n & 31]);
      } else if (MODE == 3) {
#pragma unroll
        for (int k = 0; k < 64; ++k) acc = fmaf(acc, 1.0001f, 0.5f);
      } else {
        break;
      }
      ++n;
    }
    if (acc == 12345.f) out[1000] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

template <int N, bool TS, int MODE>
void run() {
  long long* d;
  cudaMalloc(&d, 2000 * sizeof(long long));
  auto k = mma_cont<N, TS, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  const int iters = 8192;
  k<<<148, 384, 100000>>>(d, iters, nullptr);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%s N=%3d mode=%d: %.1f cycles/mma (floor %d) err=%s\n", TS ? "TS" : "SS", N, MODE,
         avg / iters, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<128, false, 0>(); run<128, false, 1>(); run<128, false, 2>(); run<128, false, 3>();
  run<64, true, 0>(); run<64, true, 1>(); run<64, true, 2>(); run<64, true, 3>();
  run<128, true, 1>(); run<128, true, 2>();
}
