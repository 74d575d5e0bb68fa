// HBM-bound fused elementwise kernels for the non-attention block of the transformer
// layer around the Ulysses path (recompute-friendly kernels that
// sp_ac re-runs in backward).  All bf16 in / bf16 out with fp32 math, 16-byte vectors,
// grid-stride loops sized to the SM count.
//   swiglu  out = silu(g) * u over gu = [g | u]        (+ backward)
//   rope    rotate-half RoPE of q/k heads with positions (rank offset applied by auto_sp)
//   ce      row-wise log-sum-exp cross entropy over bf16 logits (+ in-place gradient)
//   rms     RMSNorm forward (+ rstd) and a one-pass backward (dx and the weight gradient)
#include <cmath>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/autosp.h"
#include "rope.cuh"

extern "C" void autosp_set_error(const char* fmt, ...);

namespace autosp {
namespace fused {

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}
__device__ __forceinline__ float sigmoidf_(float x) {
  return __fdividef(1.f, 1.f + __expf(-x));  // MUFU ex2 + rcp (bf16 output: ample precision)
}

// Grid-stride walk over [rows, ffn/8] 16-byte vectors without a 64-bit division per step
// (row / column advanced incrementally), two vectors in flight per thread.
struct VecWalk {
  int64_t i, r, stride, dr;
  int c, dc, vpr;
  __device__ VecWalk(int64_t start, int64_t stride_, int vpr_) : i(start), stride(stride_), vpr(vpr_) {
    r = start / vpr;
    c = (int)(start - r * vpr);
    dr = stride / vpr;
    dc = (int)(stride - dr * vpr);
  }
  __device__ void next(int64_t& rr, int& cc) const {  // position one stride further
    rr = r + dr;
    cc = c + dc;
    if (cc >= vpr) {
      cc -= vpr;
      ++rr;
    }
  }
};

// ---------------------------------------------------------------- SwiGLU
__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out,
                                  int64_t rows, int ffn, int64_t ld_gu, int64_t ld_out) {
  const int vpr = ffn / 8;
  const int64_t total = rows * vpr;
  VecWalk w((int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x, vpr);
  while (w.i < total) {
    int64_t r2;
    int c2;
    w.next(r2, c2);
    const bool two = w.i + w.stride < total;
    const __nv_bfloat16* a = gu + w.r * ld_gu + w.c * 8;
    const __nv_bfloat16* b = gu + r2 * ld_gu + c2 * 8;
    const uint4 ga = *reinterpret_cast<const uint4*>(a);
    const uint4 ua = *reinterpret_cast<const uint4*>(a + ffn);
    uint4 gb = make_uint4(0, 0, 0, 0), ub = gb;
    if (two) {
      gb = *reinterpret_cast<const uint4*>(b);
      ub = *reinterpret_cast<const uint4*>(b + ffn);
    }
    float g[8], u[8], o[8];
    unpack8(ga, g);
    unpack8(ua, u);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = g[k] * sigmoidf_(g[k]) * u[k];
    *reinterpret_cast<uint4*>(out + w.r * ld_out + w.c * 8) = pack8(o);
    if (two) {
      unpack8(gb, g);
      unpack8(ub, u);
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = g[k] * sigmoidf_(g[k]) * u[k];
      *reinterpret_cast<uint4*>(out + r2 * ld_out + c2 * 8) = pack8(o);
    }
    w.i += 2 * w.stride;
    w.r = r2;
    w.c = c2;
    w.next(w.r, w.c);
  }
}

__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ gu,
                                  const __nv_bfloat16* __restrict__ dout,
                                  __nv_bfloat16* __restrict__ dgu, int64_t rows, int ffn,
                                  int64_t ld_gu, int64_t ld_dout, int64_t ld_dgu) {
  const int vpr = ffn / 8;
  const int64_t total = rows * vpr;
  VecWalk w((int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x, vpr);
  auto one = [&](const uint4& gv, const uint4& uv, const uint4& dv, int64_t r, int c) {
    float g[8], u[8], dy[8], dg[8], du[8];
    unpack8(gv, g);
    unpack8(uv, u);
    unpack8(dv, dy);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float sg = sigmoidf_(g[k]);
      du[k] = dy[k] * g[k] * sg;
      dg[k] = dy[k] * u[k] * sg * (1.f + g[k] * (1.f - sg));  // silu_dx (executor.py:85-88)
    }
    *reinterpret_cast<uint4*>(dgu + r * ld_dgu + c * 8) = pack8(dg);
    *reinterpret_cast<uint4*>(dgu + r * ld_dgu + ffn + c * 8) = pack8(du);
  };
  while (w.i < total) {
    int64_t r2;
    int c2;
    w.next(r2, c2);
    const bool two = w.i + w.stride < total;
    const __nv_bfloat16* a = gu + w.r * ld_gu + w.c * 8;
    const __nv_bfloat16* b = gu + r2 * ld_gu + c2 * 8;
    const uint4 ga = *reinterpret_cast<const uint4*>(a);
    const uint4 ua = *reinterpret_cast<const uint4*>(a + ffn);
    const uint4 da = *reinterpret_cast<const uint4*>(dout + w.r * ld_dout + w.c * 8);
    uint4 gb = make_uint4(0, 0, 0, 0), ub = gb, db = gb;
    if (two) {
      gb = *reinterpret_cast<const uint4*>(b);
      ub = *reinterpret_cast<const uint4*>(b + ffn);
      db = *reinterpret_cast<const uint4*>(dout + r2 * ld_dout + c2 * 8);
    }
    one(ga, ua, da, w.r, w.c);
    if (two) one(gb, ub, db, r2, c2);
    w.i += 2 * w.stride;
    w.r = r2;
    w.c = c2;
    w.next(w.r, w.c);
  }
}

// ---------------------------------------------------------------- RoPE
// x, y: [b, s, h, d] strided (d contiguous); one thread = (token, 8 rotation pairs),
// looping over every head so each angle's sincos is computed once per token.
struct RopeArgs {
  const __nv_bfloat16* x;
  __nv_bfloat16* y;
  int64_t xsb, xss, xsh, ysb, yss, ysh;
  const float* pos;  // [s] positions (already rank-offset by auto_sp)
  int b, s, h, d;
  float log2_theta;
  int inverse;       // 1: rotate by -angle (the backward)
};

__global__ void rope_kernel(const __grid_constant__ RopeArgs a) {
  const int half = a.d / 2;
  const int vpt = half / 8;  // 8-pair vectors per token
  const int64_t total = (int64_t)a.b * a.s * vpt;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(i % vpt);
    const int64_t bt = i / vpt;
    const int t = (int)(bt % a.s);
    const int bi = (int)(bt / a.s);
    const float p = a.pos[t];
    float cs[8], sn[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int j = v * 8 + k;
      const float inv_freq = exp2f(-(2.f * j / a.d) * a.log2_theta);
      sincosf(p * inv_freq, &sn[k], &cs[k]);
      if (a.inverse) sn[k] = -sn[k];
    }
    for (int hh = 0; hh < a.h; ++hh) {
      const __nv_bfloat16* xr = a.x + (int64_t)bi * a.xsb + (int64_t)t * a.xss + (int64_t)hh * a.xsh;
      __nv_bfloat16* yr = a.y + (int64_t)bi * a.ysb + (int64_t)t * a.yss + (int64_t)hh * a.ysh;
      float x1[8], x2[8], y1[8], y2[8];
      unpack8(*reinterpret_cast<const uint4*>(xr + v * 8), x1);
      unpack8(*reinterpret_cast<const uint4*>(xr + half + v * 8), x2);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        y1[k] = x1[k] * cs[k] - x2[k] * sn[k];
        y2[k] = x2[k] * cs[k] + x1[k] * sn[k];
      }
      *reinterpret_cast<uint4*>(yr + v * 8) = pack8(y1);
      *reinterpret_cast<uint4*>(yr + half + v * 8) = pack8(y2);
    }
  }
}

// Segmented RoPE: up to 3 segments (q, k rotated; v copied) in ONE launch -- the split
// of the packed QKV projection output into the attention operands (forward) and the
// assembly of the packed QKV gradient from dq/dk/dv (backward, inverse rotation), with
// no zero-filled slice_backward buffers and no adds.  One thread = (token, 8 rotation
// pairs) over every head of every segment; sincos once per (token, pair).
struct RopeSeg {
  const __nv_bfloat16* src;
  __nv_bfloat16* dst;
  int64_t ssb, sss, ssh, dsb, dss, dsh;
  int heads, rotate;
};
struct RopeSegArgs {
  RopeSeg seg[3];
  int nseg;
  const float* pos;
  int b, s, d;
  float log2_theta;
  int inverse;
};

__global__ void rope_seg_kernel(const __grid_constant__ RopeSegArgs a) {
  const int half = a.d / 2;
  const int vpt = half / 8;
  const int64_t total = (int64_t)a.b * a.s * vpt;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(i % vpt);
    const int64_t bt = i / vpt;
    const int t = (int)(bt % a.s);
    const int bi = (int)(bt / a.s);
    const float p = a.pos[t];
    float cs[8], sn[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      rope_sincos(p, v * 8 + k, a.d, a.log2_theta, &sn[k], &cs[k]);
      if (a.inverse) sn[k] = -sn[k];
    }
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      if (g >= a.nseg) break;
      const RopeSeg& S = a.seg[g];
      for (int hh = 0; hh < S.heads; ++hh) {
        const __nv_bfloat16* xr = S.src + (int64_t)bi * S.ssb + (int64_t)t * S.sss + (int64_t)hh * S.ssh;
        __nv_bfloat16* yr = S.dst + (int64_t)bi * S.dsb + (int64_t)t * S.dss + (int64_t)hh * S.dsh;
        const uint4 r1 = *reinterpret_cast<const uint4*>(xr + v * 8);
        const uint4 r2 = *reinterpret_cast<const uint4*>(xr + half + v * 8);
        if (!S.rotate) {
          *reinterpret_cast<uint4*>(yr + v * 8) = r1;
          *reinterpret_cast<uint4*>(yr + half + v * 8) = r2;
          continue;
        }
        float x1[8], x2[8], y1[8], y2[8];
        unpack8(r1, x1);
        unpack8(r2, x2);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          y1[k] = rope_lo(x1[k], x2[k], cs[k], sn[k]);
          y2[k] = rope_hi(x1[k], x2[k], cs[k], sn[k]);
        }
        *reinterpret_cast<uint4*>(yr + v * 8) = pack8(y1);
        *reinterpret_cast<uint4*>(yr + half + v * 8) = pack8(y2);
      }
    }
  }
}

// ---------------------------------------------------------------- RMSNorm
// y = x * rstd * w, rstd = 1/sqrt(mean(x^2) + eps) (reference executor.py:43-45), one warp
// per row, 16-byte vectors; the backward computes dx and the weight gradient in ONE pass
// over (dy, x): per-CTA dw partials accumulated with shared-memory reductions, then a
// small column-sum kernel (torch's path: two kernels, the weight-gradient one at ~1.6 TB/s).
constexpr int kNormThreads = 256;

// d > 4096: strided loop, x read twice (the second time from L1)
__global__ void __launch_bounds__(kNormThreads) rms_fwd_generic_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
    __nv_bfloat16* __restrict__ y, float* __restrict__ rstd, int64_t rows, int d, int64_t ldx,
    int64_t ldy, float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (kNormThreads / 32);
  const int vpr = d / 8;
  for (int64_t r = (int64_t)blockIdx.x * (kNormThreads / 32) + (threadIdx.x >> 5); r < rows;
       r += nw) {
    const __nv_bfloat16* xr = x + r * ldx;
    float ss = 0.f;
    for (int v = lane; v < vpr; v += 32) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(xr + v * 8), f);
#pragma unroll
      for (int k = 0; k < 8; ++k) ss = fmaf(f[k], f[k], ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float rs = rsqrtf(ss / d + eps);
    __nv_bfloat16* yr = y + r * ldy;
    for (int v = lane; v < vpr; v += 32) {
      float f[8], g[8];
      unpack8(*reinterpret_cast<const uint4*>(xr + v * 8), f);
      unpack8(*reinterpret_cast<const uint4*>(w + v * 8), g);
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = f[k] * rs * g[k];
      *reinterpret_cast<uint4*>(yr + v * 8) = pack8(f);
    }
    if (lane == 0) rstd[r] = rs;
  }
}

// One warp per row; lane owns VPL 16-byte vectors (v = lane + 32 i), all loaded up front
// and kept in registers for the normalising pass (no second read of x).
template <int VPL>
__global__ void __launch_bounds__(kNormThreads) rms_fwd_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
    __nv_bfloat16* __restrict__ y, float* __restrict__ rstd, int64_t rows, int d, int64_t ldx,
    int64_t ldy, float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (kNormThreads / 32);
  const int vpr = d / 8;
  for (int64_t r = (int64_t)blockIdx.x * (kNormThreads / 32) + (threadIdx.x >> 5); r < rows;
       r += nw) {
    const __nv_bfloat16* xr = x + r * ldx;
    uint4 xv[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i)
      if (lane + 32 * i < vpr) xv[i] = *reinterpret_cast<const uint4*>(xr + (lane + 32 * i) * 8);
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      if (lane + 32 * i < vpr) {
        float f[8];
        unpack8(xv[i], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) ss = fmaf(f[k], f[k], ss);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float rs = rsqrtf(ss / d + eps);
    __nv_bfloat16* yr = y + r * ldy;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int v = lane + 32 * i;
      if (v < vpr) {
        float f[8], g[8];
        unpack8(xv[i], f);
        unpack8(*reinterpret_cast<const uint4*>(w + v * 8), g);
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = f[k] * rs * g[k];
        *reinterpret_cast<uint4*>(yr + v * 8) = pack8(f);
      }
    }
    if (lane == 0) rstd[r] = rs;
  }
}

// Each lane owns VPL 16-byte column vectors (v = lane + 32 i) of every row its warp
// processes and accumulates dy * xhat for them in REGISTERS across rows; the warps of a
// CTA then combine through shared memory once (shared-memory atomics per element were
// the bottleneck of the first version).
#ifndef AUTOSP_RMS_REG
#define AUTOSP_RMS_REG 1  // keep the row's x / dy in registers between the two passes (1 CTA/SM)
#endif
template <int VPL>
__global__ void __launch_bounds__(kNormThreads, AUTOSP_RMS_REG ? 1 : 2) rms_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const __nv_bfloat16* __restrict__ w, const float* __restrict__ rstd,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ partial, int64_t rows, int d,
    int64_t lddy, int64_t ldx, int64_t lddx) {
  extern __shared__ float dw_s[];  // [d]
  for (int c = threadIdx.x; c < d; c += kNormThreads) dw_s[c] = 0.f;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * (kNormThreads / 32);
  const int vpr = d / 8;
  float acc[VPL][8];
#pragma unroll
  for (int i = 0; i < VPL; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[i][k] = 0.f;
  for (int64_t r = (int64_t)blockIdx.x * (kNormThreads / 32) + warp; r < rows; r += nw) {
    const __nv_bfloat16* xr = x + r * ldx;
    const __nv_bfloat16* gr = dy + r * lddy;
    const float rs = rstd[r];
    float dot = 0.f;  // sum_c dy*w*xhat
#if AUTOSP_RMS_REG
    uint4 xv[VPL], gv[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int v = lane + 32 * i;
      if (v < vpr) {
        xv[i] = *reinterpret_cast<const uint4*>(xr + v * 8);
        gv[i] = *reinterpret_cast<const uint4*>(gr + v * 8);
      }
    }
#endif
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int v = lane + 32 * i;
      if (v < vpr) {
        float f[8], g[8], ww[8];
#if AUTOSP_RMS_REG
        unpack8(xv[i], f);
        unpack8(gv[i], g);
#else
        unpack8(*reinterpret_cast<const uint4*>(xr + v * 8), f);
        unpack8(*reinterpret_cast<const uint4*>(gr + v * 8), g);
#endif
        unpack8(*reinterpret_cast<const uint4*>(w + v * 8), ww);
#pragma unroll
        for (int k = 0; k < 8; ++k) dot = fmaf(g[k] * ww[k], f[k] * rs, dot);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const float mdot = dot / d;
    __nv_bfloat16* dxr = dx + r * lddx;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {  // second pass: the row is L1-resident
      const int v = lane + 32 * i;
      if (v < vpr) {
        float f[8], g[8], ww[8], o8[8];
#if AUTOSP_RMS_REG
        unpack8(xv[i], f);
        unpack8(gv[i], g);
#else
        unpack8(*reinterpret_cast<const uint4*>(xr + v * 8), f);
        unpack8(*reinterpret_cast<const uint4*>(gr + v * 8), g);
#endif
        unpack8(*reinterpret_cast<const uint4*>(w + v * 8), ww);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = f[k] * rs;
          o8[k] = rs * (g[k] * ww[k] - xh * mdot);
          acc[i][k] = fmaf(g[k], xh, acc[i][k]);
        }
        *reinterpret_cast<uint4*>(dxr + v * 8) = pack8(o8);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int v = lane + 32 * i;
    if (v < vpr)
#pragma unroll
      for (int k = 0; k < 8; ++k) atomicAdd(&dw_s[v * 8 + k], acc[i][k]);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += kNormThreads) partial[(int64_t)blockIdx.x * d + c] = dw_s[c];
}

__global__ void colsum_kernel(const float* __restrict__ partial, int nb, int d,
                              __nv_bfloat16* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float acc = 0.f;
  for (int b = 0; b < nb; ++b) acc += partial[(int64_t)b * d + c];
  out[c] = __float2bfloat16_rn(acc);
}

int norm_blocks() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return (AUTOSP_RMS_REG ? 1 : 2) * sms;
}

// ---------------------------------------------------------------- cross entropy
// one CTA per row: online max/sum over the bf16 logits row, target logit gathered.
constexpr int kCeThreads = 512;

__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;
  s = s * __expf(m - mn) + s2 * __expf(m2 - mn);
  m = mn;
}

__global__ void __launch_bounds__(kCeThreads) ce_fwd_kernel(const __nv_bfloat16* __restrict__ logits,
                                                            const int64_t* __restrict__ labels,
                                                            float* __restrict__ lse,
                                                            float* __restrict__ loss, int64_t vocab,
                                                            int64_t ld) {
  const int64_t row = blockIdx.x;
  const __nv_bfloat16* x = logits + row * ld;
  float m = -INFINITY, s = 0.f;
  const int64_t nv = vocab / 8;
  // two 16-byte vectors per step (both loads in flight), one merge per 16 logits
  int64_t i = threadIdx.x;
  for (; i + blockDim.x < nv; i += 2 * blockDim.x) {
    const uint4 va = *reinterpret_cast<const uint4*>(x + i * 8);
    const uint4 vb = *reinterpret_cast<const uint4*>(x + (i + blockDim.x) * 8);
    float f[16];
    unpack8(va, *reinterpret_cast<float(*)[8]>(&f[0]));
    unpack8(vb, *reinterpret_cast<float(*)[8]>(&f[8]));
    float m8[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) m8[k] = fmaxf(fmaxf(f[k], f[k + 4]), fmaxf(f[k + 8], f[k + 12]));
    const float lm = fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3]));
    float ls = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) ls += __expf(f[k] - lm);
    online_merge(m, s, lm, ls);
  }
  for (; i < nv; i += blockDim.x) {
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(x + i * 8), f);
    float lm = f[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) lm = fmaxf(lm, f[k]);
    float ls = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) ls += __expf(f[k] - lm);
    online_merge(m, s, lm, ls);
  }
  for (int64_t i = nv * 8 + threadIdx.x; i < vocab; i += blockDim.x)
    online_merge(m, s, __bfloat162float(x[i]), 1.f);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
    online_merge(m, s, m2, s2);
  }
  __shared__ float sm[kCeThreads / 32], ss[kCeThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    sm[threadIdx.x / 32] = m;
    ss[threadIdx.x / 32] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], Ssum = ss[0];
    for (int w = 1; w < kCeThreads / 32; ++w) online_merge(M, Ssum, sm[w], ss[w]);
    const float l = M + logf(Ssum);
    lse[row] = l;
    // labels outside [0, vocab) (e.g. the -100 padding convention) are ignored: loss 0
    const int64_t lab = labels[row];
    loss[row] = (lab >= 0 && lab < vocab) ? l - __bfloat162float(x[lab]) : 0.f;
  }
}

// in place: logits -> g * (softmax - onehot(label))
__global__ void __launch_bounds__(kCeThreads) ce_bwd_kernel(__nv_bfloat16* __restrict__ logits,
                                                            const int64_t* __restrict__ labels,
                                                            const float* __restrict__ lse,
                                                            float g, int64_t vocab, int64_t ld) {
  const int64_t row = blockIdx.x;
  __nv_bfloat16* x = logits + row * ld;
  const float l = lse[row];
  const int64_t lab = labels[row];
  const int64_t nv = vocab / 8;
  if (lab < 0 || lab >= vocab) {  // ignored row: zero gradient
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x)
      *reinterpret_cast<uint4*>(x + i * 8) = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t i = nv * 8 + threadIdx.x; i < vocab; i += blockDim.x) x[i] = __float2bfloat16(0.f);
    return;
  }
  for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(x + i * 8), f);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = g * (__expf(f[k] - l) - (i * 8 + k == lab ? 1.f : 0.f));
    *reinterpret_cast<uint4*>(x + i * 8) = pack8(f);
  }
  for (int64_t i = nv * 8 + threadIdx.x; i < vocab; i += blockDim.x)
    x[i] = __float2bfloat16(g * (__expf(__bfloat162float(x[i]) - l) - (i == lab ? 1.f : 0.f)));
}

int grid_for(int64_t work, int threads) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

int launched(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    autosp_set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}

}  // namespace fused
}  // namespace autosp

using namespace autosp::fused;

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

extern "C" int autosp_swiglu_fwd(const void* gu, void* out, int64_t rows, int ffn, int64_t ld_gu,
                                 int64_t ld_out, void* stream) {
  if (!gu || !out || rows < 0 || ffn % 8 || ld_gu % 8 || ld_out % 8 || !al16(gu) || !al16(out)) {
    autosp_set_error("swiglu_fwd: pointers 16B aligned, ffn and leading dims multiples of 8");
    return AUTOSP_ERR_VALIDATION;
  }
  if (rows == 0) return AUTOSP_OK;
  const int64_t work = rows * (ffn / 8);
  swiglu_fwd_kernel<<<grid_for(work, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(gu), static_cast<__nv_bfloat16*>(out), rows, ffn, ld_gu,
      ld_out);
  return launched("swiglu_fwd");
}

extern "C" int autosp_swiglu_bwd(const void* gu, const void* dout, void* dgu, int64_t rows,
                                 int ffn, int64_t ld_gu, int64_t ld_dout, int64_t ld_dgu,
                                 void* stream) {
  if (!gu || !dout || !dgu || rows < 0 || ffn % 8 || ld_gu % 8 || ld_dout % 8 || ld_dgu % 8 ||
      !al16(gu) || !al16(dout) || !al16(dgu)) {
    autosp_set_error("swiglu_bwd: pointers 16B aligned, ffn and leading dims multiples of 8");
    return AUTOSP_ERR_VALIDATION;
  }
  if (rows == 0) return AUTOSP_OK;
  const int64_t work = rows * (ffn / 8);
  swiglu_bwd_kernel<<<grid_for(work, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(gu), static_cast<const __nv_bfloat16*>(dout),
      static_cast<__nv_bfloat16*>(dgu), rows, ffn, ld_gu, ld_dout, ld_dgu);
  return launched("swiglu_bwd");
}

extern "C" int autosp_rope(const void* x, void* y, int b, int s, int h, int d, int64_t xsb,
                           int64_t xss, int64_t xsh, int64_t ysb, int64_t yss, int64_t ysh,
                           const float* pos, float theta, int inverse, void* stream) {
  if (!x || !y || !pos || d % 16 || !al16(x) || !al16(y) || xsb % 8 || xss % 8 || xsh % 8 ||
      ysb % 8 || yss % 8 || ysh % 8 || theta <= 1.f) {
    autosp_set_error("rope: d multiple of 16, 16B-aligned views, theta > 1");
    return AUTOSP_ERR_VALIDATION;
  }
  if ((int64_t)b * s * h == 0) return AUTOSP_OK;
  RopeArgs a{static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), xsb, xss, xsh,
             ysb, yss, ysh, pos, b, s, h, d, log2f(theta), inverse};
  const int64_t work = (int64_t)b * s * (d / 16);
  rope_kernel<<<grid_for(work, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return launched("rope");
}

extern "C" int autosp_rope_segments(const autosp_rope_segment* segs, int nseg, int b, int s,
                                    int d, const float* pos, float theta, int inverse,
                                    void* stream) {
  if (!segs || nseg < 1 || nseg > 3 || !pos || d % 16 || theta <= 1.f) {
    autosp_set_error("rope_segments: 1-3 segments, d multiple of 16, theta > 1");
    return AUTOSP_ERR_VALIDATION;
  }
  RopeSegArgs a{};
  for (int g = 0; g < nseg; ++g) {
    const autosp_rope_segment& G = segs[g];
    if (!G.src || !G.dst || !al16(G.src) || !al16(G.dst) || G.src_stride_b % 8 ||
        G.src_stride_s % 8 || G.src_stride_h % 8 || G.dst_stride_b % 8 || G.dst_stride_s % 8 ||
        G.dst_stride_h % 8 || G.heads < 0) {
      autosp_set_error("rope_segments: segment %d needs 16B-aligned views", g);
      return AUTOSP_ERR_VALIDATION;
    }
    a.seg[g] = RopeSeg{static_cast<const __nv_bfloat16*>(G.src), static_cast<__nv_bfloat16*>(G.dst),
                       G.src_stride_b, G.src_stride_s, G.src_stride_h, G.dst_stride_b,
                       G.dst_stride_s, G.dst_stride_h, G.heads, G.rotate};
  }
  if ((int64_t)b * s == 0) return AUTOSP_OK;
  a.nseg = nseg;
  a.pos = pos;
  a.b = b;
  a.s = s;
  a.d = d;
  a.log2_theta = log2f(theta);
  a.inverse = inverse;
  const int64_t work = (int64_t)b * s * (d / 16);
  rope_seg_kernel<<<grid_for(work, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return launched("rope_segments");
}

extern "C" int autosp_rms_norm_fwd(const void* x, const void* w, void* y, float* rstd,
                                   int64_t rows, int d, int64_t ld_x, int64_t ld_y, float eps,
                                   void* stream) {
  if (!x || !w || !y || !rstd || d % 8 || d < 8 || !al16(x) || !al16(w) || !al16(y) ||
      ld_x % 8 || ld_y % 8) {
    autosp_set_error("rms_norm_fwd: d multiple of 8, 16B-aligned rows");
    return AUTOSP_ERR_VALIDATION;
  }
  if (rows == 0) return AUTOSP_OK;
  const int64_t warps = rows;
  auto go = [&](auto kern) {
    kern<<<grid_for(warps * 32, kNormThreads), kNormThreads, 0,
           static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
        static_cast<__nv_bfloat16*>(y), rstd, rows, d, ld_x, ld_y, eps);
  };
  const int vpl = (d / 8 + 31) / 32;
  if (vpl <= 1) go(rms_fwd_kernel<1>);
  else if (vpl <= 2) go(rms_fwd_kernel<2>);
  else if (vpl <= 4) go(rms_fwd_kernel<4>);
  else if (vpl <= 8) go(rms_fwd_kernel<8>);
  else if (vpl <= 16) go(rms_fwd_kernel<16>);
  else go(rms_fwd_generic_kernel);
  return launched("rms_norm_fwd");
}

extern "C" size_t autosp_rms_norm_bwd_workspace_bytes(int d) {
  return (size_t)norm_blocks() * d * sizeof(float);
}

extern "C" int autosp_rms_norm_bwd(const void* dy, const void* x, const void* w,
                                   const float* rstd, void* dx, void* dw, void* workspace,
                                   int64_t rows, int d, int64_t ld_dy, int64_t ld_x,
                                   int64_t ld_dx, void* stream) {
  if (!dy || !x || !w || !rstd || !dx || !dw || !workspace || d % 8 || d < 8 ||
      d > 4096 || !al16(dy) || !al16(x) || !al16(w) || !al16(dx) ||
      ld_dy % 8 || ld_x % 8 || ld_dx % 8) {
    autosp_set_error("rms_norm_bwd: d multiple of 8 (<= 4096), 16B-aligned rows");
    return AUTOSP_ERR_VALIDATION;
  }
  const int nb = norm_blocks();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t smem = (size_t)d * sizeof(float);
  const int vpl = (d / 8 + 31) / 32;  // 16-byte vectors per lane
  auto go = [&](auto kern) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<nb, kNormThreads, smem, st>>>(
        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x),
        static_cast<const __nv_bfloat16*>(w), rstd, static_cast<__nv_bfloat16*>(dx),
        static_cast<float*>(workspace), rows, d, ld_dy, ld_x, ld_dx);
  };
  if (vpl <= 1) go(rms_bwd_kernel<1>);
  else if (vpl <= 2) go(rms_bwd_kernel<2>);
  else if (vpl <= 4) go(rms_bwd_kernel<4>);
  else if (vpl <= 8) go(rms_bwd_kernel<8>);
  else if (vpl <= 16) go(rms_bwd_kernel<16>);
  else {
    autosp_set_error("rms_norm_bwd: d = %d > 4096 unsupported", d);
    return AUTOSP_ERR_UNSUPPORTED;
  }
  colsum_kernel<<<(d + 255) / 256, 256, 0, st>>>(static_cast<const float*>(workspace), nb, d,
                                                 static_cast<__nv_bfloat16*>(dw));
  return launched("rms_norm_bwd");
}

extern "C" int autosp_ce_fwd(const void* logits, const int64_t* labels, float* lse, float* loss,
                             int64_t rows, int64_t vocab, int64_t ld, void* stream) {
  if (!logits || !labels || !lse || !loss || ld % 8 || !al16(logits) || vocab < 1) {
    autosp_set_error("ce_fwd: logits 16B aligned with leading dim multiple of 8");
    return AUTOSP_ERR_VALIDATION;
  }
  if (rows == 0) return AUTOSP_OK;
  ce_fwd_kernel<<<(unsigned)rows, kCeThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(logits), labels, lse, loss, vocab, ld);
  return launched("ce_fwd");
}

extern "C" int autosp_ce_bwd(void* logits, const int64_t* labels, const float* lse, float g,
                             int64_t rows, int64_t vocab, int64_t ld, void* stream) {
  if (!logits || !labels || !lse || ld % 8 || !al16(logits) || vocab < 1) {
    autosp_set_error("ce_bwd: logits 16B aligned with leading dim multiple of 8");
    return AUTOSP_ERR_VALIDATION;
  }
  if (rows == 0) return AUTOSP_OK;
  ce_bwd_kernel<<<(unsigned)rows, kCeThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<__nv_bfloat16*>(logits), labels, lse, g, vocab, ld);
  return launched("ce_bwd");
}

int autosp_preload_fused() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, swiglu_fwd_kernel);
  cudaFuncGetAttributes(&a, swiglu_bwd_kernel);
  cudaFuncGetAttributes(&a, rope_kernel);
  cudaFuncGetAttributes(&a, rope_seg_kernel);
  cudaFuncGetAttributes(&a, rms_fwd_kernel<8>);
  cudaFuncGetAttributes(&a, rms_fwd_kernel<16>);
  cudaFuncGetAttributes(&a, rms_bwd_kernel<8>);
  cudaFuncGetAttributes(&a, rms_bwd_kernel<16>);
  cudaFuncGetAttributes(&a, colsum_kernel);
  cudaFuncGetAttributes(&a, ce_fwd_kernel);
  cudaFuncGetAttributes(&a, ce_bwd_kernel);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

// ---------------------------------------------------------------- AdamW (bf16 params/state)
// One launch updates up to kAdamwMaxT tensors: block b works on 2048 elements of the
// tensor whose chunk range holds b (binary search over the chunk prefix).  Math in fp32,
// the same sequence as torch's AdamW: p *= 1 - lr*wd; m = lerp(m, g, 1-b1);
// v = b2*v + (1-b2)*g^2; p -= lr/bc1 * m / (sqrt(v)/sqrt(bc2) + eps).
namespace adamw_impl {
constexpr int kAdamwMaxT = 64;
constexpr int kAdamwThreads = 256;
constexpr int kAdamwChunk = kAdamwThreads * 8;
struct AdamwArgs {
  __nv_bfloat16* p[kAdamwMaxT];
  const __nv_bfloat16* g[kAdamwMaxT];
  __nv_bfloat16* m[kAdamwMaxT];
  __nv_bfloat16* v[kAdamwMaxT];
  int64_t n[kAdamwMaxT];
  int64_t chunk0[kAdamwMaxT + 1];  // prefix of chunk counts
  int count;
  float lr, b1, b2, eps, decay, step_size, inv_sqrt_bc2;
};

__device__ __forceinline__ void adamw_one(float& p, float g, float& m, float& v,
                                          const AdamwArgs& a) {
  p *= a.decay;
  m = m + (1.f - a.b1) * (g - m);
  v = a.b2 * v + (1.f - a.b2) * g * g;
  p -= a.step_size * m / (sqrtf(v) * a.inv_sqrt_bc2 + a.eps);
}

__global__ void __launch_bounds__(kAdamwThreads) adamw_bf16_kernel(const __grid_constant__ AdamwArgs a) {
  const int64_t blk = blockIdx.x;
  int lo = 0, hi = a.count - 1;  // last t with chunk0[t] <= blk
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.chunk0[mid] <= blk) lo = mid;
    else hi = mid - 1;
  }
  const int t = lo;
  const int64_t e0 = (blk - a.chunk0[t]) * kAdamwChunk + threadIdx.x * 8;
  const int64_t n = a.n[t];
  if (e0 >= n) return;
  __nv_bfloat16* P = a.p[t] + e0;
  const __nv_bfloat16* G = a.g[t] + e0;
  __nv_bfloat16* M = a.m[t] + e0;
  __nv_bfloat16* V = a.v[t] + e0;
  const bool vec = e0 + 8 <= n && ((reinterpret_cast<uintptr_t>(P) | reinterpret_cast<uintptr_t>(G) |
                                     reinterpret_cast<uintptr_t>(M) | reinterpret_cast<uintptr_t>(V)) & 15) == 0;
  if (vec) {
    float p[8], g[8], m[8], v[8];
    unpack8(*reinterpret_cast<const uint4*>(P), p);
    unpack8(*reinterpret_cast<const uint4*>(G), g);
    unpack8(*reinterpret_cast<const uint4*>(M), m);
    unpack8(*reinterpret_cast<const uint4*>(V), v);
#pragma unroll
    for (int k = 0; k < 8; ++k) adamw_one(p[k], g[k], m[k], v[k], a);
    *reinterpret_cast<uint4*>(P) = pack8(p);
    *reinterpret_cast<uint4*>(M) = pack8(m);
    *reinterpret_cast<uint4*>(V) = pack8(v);
  } else {
    for (int k = 0; k < 8 && e0 + k < n; ++k) {
      float p = __bfloat162float(P[k]), g = __bfloat162float(G[k]);
      float m = __bfloat162float(M[k]), v = __bfloat162float(V[k]);
      adamw_one(p, g, m, v, a);
      P[k] = __float2bfloat16_rn(p);
      M[k] = __float2bfloat16_rn(m);
      V[k] = __float2bfloat16_rn(v);
    }
  }
}
}  // namespace adamw_impl

extern "C" int autosp_adamw_bf16(const autosp_adamw_tensor* tensors, int count, float lr,
                                 float beta1, float beta2, float eps, float weight_decay, int step,
                                 void* stream) {
  if ((count > 0 && !tensors) || count < 0 || step < 1) {
    autosp_set_error("adamw_bf16: bad arguments (count %d, step %d)", count, step);
    return AUTOSP_ERR_VALIDATION;
  }
  const float bc1 = 1.f - powf(beta1, (float)step), bc2 = 1.f - powf(beta2, (float)step);
  // each launch packs the next (up to) 64 NON-EMPTY tensors; `next` is the first tensor
  // not yet packed, so empty tensors are skipped without updating any tensor twice
  for (int next = 0; next < count;) {
    adamw_impl::AdamwArgs a{};
    a.count = 0;
    int64_t chunks = 0;
    for (; next < count && a.count < adamw_impl::kAdamwMaxT; ++next) {
      const int i = next;
      const autosp_adamw_tensor& t = tensors[i];
      if (t.n <= 0) continue;
      if (!t.p || !t.g || !t.m || !t.v) {
        autosp_set_error("adamw_bf16: tensor %d has a null pointer", i);
        return AUTOSP_ERR_VALIDATION;
      }
      const int j = a.count++;
      a.p[j] = static_cast<__nv_bfloat16*>(t.p);
      a.g[j] = static_cast<const __nv_bfloat16*>(t.g);
      a.m[j] = static_cast<__nv_bfloat16*>(t.m);
      a.v[j] = static_cast<__nv_bfloat16*>(t.v);
      a.n[j] = t.n;
      a.chunk0[j] = chunks;
      chunks += (t.n + adamw_impl::kAdamwChunk - 1) / adamw_impl::kAdamwChunk;
    }
    if (a.count == 0) continue;
    a.chunk0[a.count] = chunks;
    a.lr = lr;
    a.b1 = beta1;
    a.b2 = beta2;
    a.eps = eps;
    a.decay = 1.f - lr * weight_decay;
    a.step_size = lr / bc1;
    a.inv_sqrt_bc2 = 1.f / sqrtf(bc2);
    adamw_impl::adamw_bf16_kernel<<<(unsigned)chunks, adamw_impl::kAdamwThreads, 0,
                               static_cast<cudaStream_t>(stream)>>>(a);
    const int rc = launched("adamw_bf16");
    if (rc) return rc;
  }
  return AUTOSP_OK;
}
