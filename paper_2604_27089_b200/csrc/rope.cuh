// Rotate-half RoPE math shared by the segmented RoPE kernel (fused.cu) and the RoPE-fused
// all-to-all push (a2a.cu), so both produce bit-identical results.
#pragma once
#include <cmath>

namespace autosp {

// angle of rotation pair j (0 <= j < d/2) at position p: p * theta^(-2j/d)
__device__ __forceinline__ void rope_sincos(float p, int j, int d, float log2_theta,
                                            float* sn, float* cs) {
  const float inv_freq = exp2f(-(2.f * j / d) * log2_theta);
  sincosf(p * inv_freq, sn, cs);
}
// first half element x1 with partner x2: x1 c - x2 s; second half x2: x2 c + x1 s.
// The rounding is pinned with explicit intrinsics (one product rounded, then one fma):
// left to the compiler, the FMA contraction of a*b + c*d depends on the surrounding code,
// and the kernels sharing this math (segmented RoPE, K1's RoPE push, K0's epilogue) must
// agree bit for bit.
__device__ __forceinline__ float rope_lo(float x1, float x2, float c, float s) {
  return __fmaf_rn(x1, c, __fmul_rn(-x2, s));
}
__device__ __forceinline__ float rope_hi(float x1, float x2, float c, float s) {
  return __fmaf_rn(x2, c, __fmul_rn(x1, s));
}

}  // namespace autosp
