// TMEM read throughput on sm_100a: W warps of one CTA per SM repeatedly issue
// tcgen05.ld.sync.aligned.32x32b.x32 (32 lanes x 32 columns x 4 B = 4 KB per warp
// instruction) + tcgen05.wait::ld, and we report bytes / clock / SM (development
// microbenchmark; not part of the library).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_27089_b200/csrc/ptx.cuh"
using namespace autosp;

AUTOSP_DEV void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,"
      "%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,"
      "%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]),
        "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]),
        "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),
        "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]),
        "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}
// 16x256b: 16 lanes x 256 bits per "x1"; x8 -> 4 KB per warp instruction like 32x32b.x32
AUTOSP_DEV void tmem_ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

template <int MODE>  // 0: 32x32b.x64, 1: 16x256b.x8
__global__ void tmem_ld_shape(long long* cyc, float* sink, int iters) {
  __shared__ uint32_t tm;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tm);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + ((warp / 4) * 64) % 512;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      uint32_t r[64];
      tmem_ld64(base, r);
      tmem_wait_ld();
      acc += __uint_as_float(r[0]) + __uint_as_float(r[63]);
    } else {
      uint32_t r[32], r2[32];
      tmem_ld_16x256b_x8(base, r);
      tmem_ld_16x256b_x8(base + (16u << 16), r2);
      tmem_wait_ld();
      acc += __uint_as_float(r[0]) + __uint_as_float(r2[31]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

template <int NLD>
__global__ void tmem_ld_rate(long long* cyc, float* sink, int iters) {
  __shared__ uint32_t tm;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tm);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tm + ((uint32_t)((warp & 3) * 32) << 16) + (warp / 4) * 32 % 512;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[NLD][32];
#pragma unroll
    for (int k = 0; k < NLD; ++k) tmem_ld32(base + (k * 64) % 512, r[k]);
    tmem_wait_ld();
#pragma unroll
    for (int k = 0; k < NLD; ++k) acc += __uint_as_float(r[k][0]) + __uint_as_float(r[k][31]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(float));
  const int iters = 2000;
  for (int warps : {1, 2, 4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      tmem_ld_rate<2><<<148, warps * 32>>>(cyc, sink, iters);
      cudaDeviceSynchronize();
    }
    long long h;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = (double)warps * iters * 2 * 4096;
    printf("warps %2d, 2 x ld.32x32b.x32 per wait: %.1f B/clk/SM (%lld cycles)\n", warps,
           bytes / h, h);
  }
  for (int warps : {4, 8, 16}) {
    tmem_ld_rate<4><<<148, warps * 32>>>(cyc, sink, iters);
    cudaDeviceSynchronize();
    tmem_ld_rate<4><<<148, warps * 32>>>(cyc, sink, iters);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = (double)warps * iters * 4 * 4096;
    printf("warps %2d, 4 x ld.32x32b.x32 per wait: %.1f B/clk/SM (%lld cycles)\n", warps,
           bytes / h, h);
  }
  for (int warps : {1, 4, 8}) {  // (16 warps x 64 registers of x64 exceed the launch)
    long long h;
    tmem_ld_shape<0><<<148, warps * 32>>>(cyc, sink, iters);
    tmem_ld_shape<0><<<148, warps * 32>>>(cyc, sink, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warps %2d, 1 x ld.32x32b.x64 per wait: %.1f B/clk/SM\n", warps,
           (double)warps * iters * 8192 / h);
    tmem_ld_shape<1><<<148, warps * 32>>>(cyc, sink, iters);
    tmem_ld_shape<1><<<148, warps * 32>>>(cyc, sink, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warps %2d, 2 x ld.16x256b.x8 per wait: %.1f B/clk/SM\n", warps,
           (double)warps * iters * 8192 / h);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
