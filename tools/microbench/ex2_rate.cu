// MUFU exp2 throughput on sm_100a: ex2.approx.ftz.f32 (one result per instruction) vs
// ex2.approx.ftz.bf16x2 (two results per instruction), plus the accuracy of the packed
// form against exp2f on the attention softmax's input range (development microbenchmark;
// not part of the library).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2_f32(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

constexpr int kChains = 8;

// each thread runs kChains independent dependency chains of `iters` exps
__global__ void rate_f32(float* out, int iters, long long* cyc) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = -0.001f * (threadIdx.x + c);
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = ex2_f32(v[c]) - 1.0f;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void rate_bf16x2(float* out, int iters, long long* cyc) {
  uint32_t v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = 0xBC00BC00u + threadIdx.x + c;  // ~ -0.0078
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = ex2_bf16x2(v[c]) ^ 0x80008000u;  // negate
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += __uint_as_float(v[c] << 16);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// accuracy: bf16x2 exp2 of bf16(x) vs exp2f(x) for x in [-30, 0]
__global__ void accuracy(float* maxabs, float* maxrel_big, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x = -30.0f * i / (n - 1);
  __nv_bfloat162 xb = __floats2bfloat162_rn(x, x);
  uint32_t y = ex2_bf16x2(*reinterpret_cast<uint32_t*>(&xb));
  float yb = __uint_as_float(y << 16);
  float ref = exp2f(x);
  float ae = fabsf(yb - ref);
  atomicMax(reinterpret_cast<int*>(maxabs), __float_as_int(ae));
  if (ref > 1e-2f) atomicMax(reinterpret_cast<int*>(maxrel_big), __float_as_int(ae / ref));
}

int main() {
  const int blocks = 148 * 4, threads = 256, iters = 4096;
  float* out;
  long long* cyc;
  cudaMalloc(&out, blocks * threads * sizeof(float));
  cudaMalloc(&cyc, blocks * sizeof(long long));
  long long h[4];
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms32, ms16;
    cudaEventRecord(a);
    rate_f32<<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms32, a, b);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long c32 = h[0];
    cudaEventRecord(a);
    rate_bf16x2<<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms16, a, b);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long c16 = h[0];
    double n_inst = (double)blocks * threads * iters * kChains;
    // per SM: 4 resident blocks x 256 threads; instructions per clock per SM
    double per_sm = 4.0 * threads * iters * kChains;
    printf("rep %d: f32 ex2: %.3f ms, %.2f inst/clk/SM (%.1f Gexp/s) | bf16x2 ex2: %.3f ms, "
           "%.2f inst/clk/SM (%.1f Gexp/s, 2 results/inst)\n",
           rep, ms32, per_sm / c32, n_inst / ms32 / 1e6, ms16, per_sm / c16,
           2 * n_inst / ms16 / 1e6);
  }
  float *ma, *mr;
  cudaMalloc(&ma, 4);
  cudaMalloc(&mr, 4);
  cudaMemset(ma, 0, 4);
  cudaMemset(mr, 0, 4);
  const int n = 1 << 20;
  accuracy<<<(n + 255) / 256, 256>>>(ma, mr, n);
  float hma, hmr;
  cudaMemcpy(&hma, ma, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hmr, mr, 4, cudaMemcpyDeviceToHost);
  printf("bf16x2 ex2 of bf16(x), x in [-30,0]: max abs err %.3e, max rel err (ref > 1e-2) %.3e\n",
         hma, hmr);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
