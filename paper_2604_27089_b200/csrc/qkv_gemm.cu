// K0: the packed QKV projection of the Llama block, Y = X W^T (bf16 in, fp32 accumulate in
// TMEM), with the seq->head all-to-all (K1) folded into its epilogue: every output row of a
// (token, head) pair is rounded to bf16, RoPE-rotated if it is a q/k head (positions of this
// rank's tokens, the rotate-half math shared with K1 through rope.cuh, so the result is
// bit-identical to "GEMM -> bf16 -> K1"), and stored straight into the head owner's receive
// region in the attention layout [b, h/P, s, d] (reference semantics: the projection
// Linear of transformer.py:66-72 followed by all_to_all_shards("seq_to_head"),
// executor.py:203-230).  The reshard therefore overlaps the GEMM tile by tile instead of
// being a separate pass that re-reads the projection output.
//
// sm_100a design:
//  * persistent: one CTA per SM walks the (128-token x 256-column) output tiles;
//  * warp 0: TMA producer, a 4-stage ring of {X tile 128x64, W tile 256x64} (128B swizzle);
//  * warp 1: tcgen05.mma issuer (M=128, N=256, K=16, both operands K-major), TMEM owner;
//    two 256-column fp32 accumulators, so the epilogue of tile i overlaps the mainloop of
//    tile i+1;
//  * warps 2-5: epilogue, thread = token row (TMEM lane); each (token, head) row goes out
//    through a swizzled shared-memory staging area so a warp stores its 32 tokens -- which
//    are consecutive in the head-major destination -- as one contiguous 32*d*2-byte block
//    (512 bytes per store instruction: full lines for NVLink and HBM alike);
//  * push = 0: plain GEMM into a local row-major Y (no RoPE) -- the unfused reference path.
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/autosp.h"
#include "flags.cuh"
#include "ptx.cuh"
#include "rope.cuh"
#include "tma.cuh"

extern "C" void autosp_set_error(const char* fmt, ...);
int autosp_internal_handshake(uint32_t* const* flags, int world, int rank, uint32_t epoch,
                              cudaStream_t stream);

namespace autosp {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int kStages = 4;
constexpr int A_TILE = BM * BK * 2;
constexpr int B_TILE = BN * BK * 2;
constexpr int STAGE = A_TILE + B_TILE;
constexpr int kThreads = 6 * 32;
constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2;
constexpr int STAGING = 4 * 32 * 256;  // 4 warps x 32 rows x (up to) 256 B
constexpr int BAR_OFF = kStages * STAGE + STAGING;
constexpr int SMEM = BAR_OFF + 256 + 1024;  // + alignment slack
static_assert(SMEM <= 232448, "shared memory budget");

struct Params {
  CUtensorMap tm_a, tm_b;
  int M, N, K;
  int s_loc;        // tokens per batch element of X (rows m = b * s_loc + t)
  int hq, hkv, d;   // global head counts of the packed output, head_dim
  const float* pos; // RoPE positions of this rank's tokens [s_loc]
  float log2_theta;
  int rope;
  int push, P, rank, S;
  int64_t dst_off[3];  // q / k / v destination offsets (bytes) in every receive region
  char* peer_base[AUTOSP_MAX_WORLD];
  uint32_t* peer_flags[AUTOSP_MAX_WORLD];
  uint32_t epoch, check;
  __nv_bfloat16* y;  // push == 0
  int64_t ldy;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1) qkv_gemm_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* full = bars;                  // [kStages]
  uint64_t* empty = full + kStages;       // [kStages]
  uint64_t* acc_full = empty + kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = warp_id();
  const int lane = lane_id();
  const int n_tiles_n = p.N / BN;
  const int n_tiles = (p.M / BM) * n_tiles_n;
  const int n_kb = p.K / BK;

  if (warp == kTmaWarp && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, 4);  // one arrival per epilogue warp
    }
    fence_mbar_init();
    tma_prefetch_desc(&p.tm_a);
    tma_prefetch_desc(&p.tm_b);
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == kTmaWarp) {
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();  // W tiles are re-read by every m tile
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int m0 = (tile / n_tiles_n) * BM, n0 = (tile % n_tiles_n) * BN;
        for (int kb = 0; kb < n_kb; ++kb, ++it) {
          const int st = it % kStages;
          mbar_wait(empty + st, ((it / kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(full + st, STAGE);
          uint8_t* sa = smem + st * STAGE;
          tma_load_4d(sa, &p.tm_a, full + st, kb * BK, m0, 0, 0, pol_a);
          tma_load_4d(sa + A_TILE, &p.tm_b, full + st, kb * BK, n0, 0, 0, pol_b);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    constexpr uint32_t idesc = make_idesc_bf16(BM, BN, 0, 0);
    int it = 0, lt = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++lt) {
      const int buf = lt & 1;
      mbar_wait(acc_empty + buf, ((lt >> 1) & 1) ^ 1);  // the epilogue drained this buffer
      tc_fence_after();
      const uint32_t acc = tmem + buf * BN;
      for (int kb = 0; kb < n_kb; ++kb, ++it) {
        const int st = it % kStages;
        mbar_wait(full + st, (it / kStages) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + st * STAGE);
        const uint64_t da = make_smem_desc(sa, 16, 1024, 2);
        const uint64_t db = make_smem_desc(sa + A_TILE, 16, 1024, 2);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)  // +32 B per K-step inside the 128B atom
            mma_ss(acc, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), idesc,
                   (kb | kk) != 0);
          tc_commit(empty + st);
          if (kb == n_kb - 1) tc_commit(acc_full + buf);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    constexpr int ROWB = D * 2;        // bytes of one (token, head) row
    constexpr int VPR = ROWB / 16;     // 16-byte units per row
    constexpr int HPT = BN / D;        // heads per tile
    const int quarter = warp & 3;      // TMEM lanes [32q, 32q + 32)
    const int row = quarter * 32 + lane;
    uint8_t* stage = smem + kStages * STAGE + (warp - kEpiWarp0) * (32 * ROWB);
    const int H3 = p.hq + 2 * p.hkv;
    int lt = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++lt) {
      const int buf = lt & 1;
      const int m0 = (tile / n_tiles_n) * BM, n0 = (tile % n_tiles_n) * BN;
      mbar_wait(acc_full + buf, (lt >> 1) & 1);
      tc_fence_after();
      const int m = m0 + row;
      const int bi = m / p.s_loc, t = m - bi * p.s_loc;
      const float tp = p.rope ? __ldg(p.pos + t) : 0.f;
      const uint32_t acc = tmem + ((uint32_t)(quarter * 32) << 16) + buf * BN;
      // d <= 64: the token's rotation angles are shared by every q/k head of the tile --
      // computed once per tile (same rope_sincos calls as K1: bit-identical values)
      constexpr bool kHoist = D <= 64;
      float rs[kHoist ? D / 2 : 1], rc[kHoist ? D / 2 : 1];
      if constexpr (kHoist) {
        if (p.rope && n0 / D < p.hq + p.hkv) {
#pragma unroll
          for (int j = 0; j < D / 2; ++j) rope_sincos(tp, j, D, p.log2_theta, &rs[j], &rc[j]);
        }
      }
#pragma unroll 1
      for (int hh = 0; hh < HPT; ++hh) {
        const int gh = n0 / D + hh;  // head in the packed [hq | hkv | hkv] order
        uint32_t v[D / 2];           // the row as bf16 pairs
        {
          uint32_t x[32];
#pragma unroll
          for (int c = 0; c < D; c += 32) {
            tmem_ld32(acc + hh * D + c, x);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i)
              v[c / 2 + i] = pack_bf16(__uint_as_float(x[2 * i]), __uint_as_float(x[2 * i + 1]));
          }
        }
        if (p.rope && gh < p.hq + p.hkv) {
          // rotate-half on the bf16-rounded row (exactly what K1 does to the stored Y)
#pragma unroll
          for (int i = 0; i < D / 4; ++i) {  // pairs (j, j + D/2) for j = 2i, 2i + 1
            const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&v[i]);
            const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&v[D / 4 + i]);
            const float2 l2 = __bfloat1622float2(lo), h2 = __bfloat1622float2(hi);
            float s0, c0, s1, c1;
            if constexpr (kHoist) {
              s0 = rs[2 * i], c0 = rc[2 * i], s1 = rs[2 * i + 1], c1 = rc[2 * i + 1];
            } else {
              rope_sincos(tp, 2 * i, D, p.log2_theta, &s0, &c0);
              rope_sincos(tp, 2 * i + 1, D, p.log2_theta, &s1, &c1);
            }
            const __nv_bfloat162 nlo = __floats2bfloat162_rn(rope_lo(l2.x, h2.x, c0, s0),
                                                             rope_lo(l2.y, h2.y, c1, s1));
            const __nv_bfloat162 nhi = __floats2bfloat162_rn(rope_hi(l2.x, h2.x, c0, s0),
                                                             rope_hi(l2.y, h2.y, c1, s1));
            v[i] = *reinterpret_cast<const uint32_t*>(&nlo);
            v[D / 4 + i] = *reinterpret_cast<const uint32_t*>(&nhi);
          }
        }
        if (!p.push) {  // plain GEMM output, row-major [M, N]
          uint4* dst = reinterpret_cast<uint4*>(p.y + (int64_t)m * p.ldy + n0 + hh * D);
#pragma unroll
          for (int u = 0; u < VPR; ++u)
            dst[u] = make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
          continue;
        }
        // stage the warp's 32 rows (16-byte units XOR-swizzled by row), then store them as
        // one contiguous block: consecutive tokens are consecutive rows of the head-major
        // destination [b, Ht/P, S, d] (s_loc % 128 == 0, so a warp never straddles a batch)
        __syncwarp();
#pragma unroll
        for (int u = 0; u < VPR; ++u)
          sts128(stage + lane * ROWB + ((u ^ (lane & 7)) << 4),
                 make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]));
        __syncwarp();
        const int tsel = gh < p.hq ? 0 : (gh < p.hq + p.hkv ? 1 : 2);
        const int Ht = tsel == 0 ? p.hq : p.hkv;
        const int lh = gh - (tsel == 0 ? 0 : (tsel == 1 ? p.hq : p.hq + p.hkv));
        const int hl_per = Ht / p.P;
        const int j = lh / hl_per, hl = lh - j * hl_per;
        const int mw = m0 + quarter * 32;  // the warp's first token
        const int bw = mw / p.s_loc, tw = mw - bw * p.s_loc;
        char* dst = p.peer_base[j] + p.dst_off[tsel] +
                    ((((int64_t)bw * hl_per + hl) * p.S) + (int64_t)p.rank * p.s_loc + tw) * ROWB;
#pragma unroll
        for (int k = 0; k < VPR; ++k) {
          const int i = k * 32 + lane;  // 16-byte unit of the 32-row block
          const int r = i / VPR, u = i % VPR;
          *reinterpret_cast<uint4*>(dst + (int64_t)i * 16) =
              lds128u(stage + r * ROWB + ((u ^ (r & 7)) << 4));
        }
      }
      tc_fence_before();
      mbar_arrive_warp(acc_empty + buf);
    }
    (void)H3;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
  if (p.push) publish_arrival(p.peer_flags, p.P, p.rank, p.epoch, p.check, gridDim.x);
}

// 2-D bf16 map over a row-major [rows, cols] matrix with leading dimension ld (elements),
// box {64, box_rows}, 128B swizzle (expressed as a 4-D map with unit outer dims).
inline bool make_map_rowmajor(CUtensorMap* map, const void* ptr, int rows, int cols, int64_t ld,
                              int box_rows) {
  return make_map_bhsd(map, ptr, 1, 1, rows, cols, (int64_t)rows * ld, (int64_t)rows * ld, ld,
                       BK, box_rows, 128);
}

}  // namespace gemm
}  // namespace autosp

extern "C" int autosp_qkv_gemm(const void* x, int64_t ldx, const void* w, int64_t ldw, int M,
                               int K, int hq, int hkv, int d, int s_loc, const float* pos,
                               float theta, int rope, void* y, int64_t ldy,
                               const autosp_a2a_tensor* dst3, int world, int rank,
                               void* const* peer_base, uint32_t* const* peer_flags,
                               uint32_t epoch, void* stream) {
  using namespace autosp::gemm;
  const int N = (hq + 2 * hkv) * d;
  if (!x || !w || M < 1 || K < 1 || hq < 1 || hkv < 1 || (d != 32 && d != 64 && d != 128)) {
    autosp_set_error("qkv_gemm: bad arguments (M=%d K=%d hq=%d hkv=%d d=%d)", M, K, hq, hkv, d);
    return AUTOSP_ERR_VALIDATION;
  }
  if (M % BM || N % BN || K % BK || s_loc < 1 || s_loc % BM || M % s_loc) {
    autosp_set_error("qkv_gemm: needs M %% 128 == 0, s_loc %% 128 == 0, (hq+2hkv)*d %% 256 == 0 "
                     "and K %% 64 == 0 (M=%d s_loc=%d N=%d K=%d)", M, s_loc, N, K);
    return AUTOSP_ERR_UNSUPPORTED;
  }
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15 || ldx % 8 ||
      ldw % 8) {
    autosp_set_error("qkv_gemm: X / W must be 16-byte aligned with 16-byte row strides");
    return AUTOSP_ERR_VALIDATION;
  }
  if (rope && (!pos || theta <= 1.f)) {
    autosp_set_error("qkv_gemm: rope needs positions and theta > 1");
    return AUTOSP_ERR_VALIDATION;
  }
  Params p{};
  if (!make_map_rowmajor(&p.tm_a, x, M, K, ldx, BM) ||
      !make_map_rowmajor(&p.tm_b, w, N, K, ldw, BN)) {
    autosp_set_error("qkv_gemm: cuTensorMapEncodeTiled failed");
    return AUTOSP_ERR_VALIDATION;
  }
  p.M = M;
  p.N = N;
  p.K = K;
  p.s_loc = s_loc;
  p.hq = hq;
  p.hkv = hkv;
  p.d = d;
  p.pos = pos;
  p.rope = rope ? 1 : 0;
  p.log2_theta = rope ? log2f(theta) : 0.f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dst3) {  // fused seq->head push
    if (world < 1 || world > AUTOSP_MAX_WORLD || rank < 0 || rank >= world || !peer_base ||
        !peer_flags || hq % world || hkv % world) {
      autosp_set_error("qkv_gemm: bad push arguments (world %d rank %d hq %d hkv %d)", world,
                       rank, hq, hkv);
      return AUTOSP_ERR_VALIDATION;
    }
    p.push = 1;
    p.P = world;
    p.rank = rank;
    p.S = s_loc * world;
    for (int i = 0; i < 3; ++i) {
      const int Ht = i == 0 ? hq : hkv;
      const autosp_a2a_tensor& t = dst3[i];
      // destination must be the contiguous head-major [b, Ht/P, S, d] attention operand
      if (t.dst_offset % 16 || t.dst_stride_s != d || t.dst_stride_h != (int64_t)p.S * d ||
          t.dst_stride_b != (int64_t)(Ht / world) * p.S * d || t.heads != Ht) {
        autosp_set_error("qkv_gemm: destination %d must be contiguous [b, h/P, S, d]", i);
        return AUTOSP_ERR_VALIDATION;
      }
      p.dst_off[i] = t.dst_offset;
    }
    for (int j = 0; j < world; ++j) {
      if (!peer_base[j] || !peer_flags[j]) {
        autosp_set_error("qkv_gemm: peer %d base/flags null", j);
        return AUTOSP_ERR_VALIDATION;
      }
      p.peer_base[j] = static_cast<char*>(peer_base[j]);
      p.peer_flags[j] = peer_flags[j];
    }
    p.epoch = epoch;
    p.check = autosp_a2a_check(AUTOSP_SEQ_TO_HEAD, dst3, 3);
    if (world > 1) {
      int rc = autosp_internal_handshake(p.peer_flags, world, rank, epoch, st);
      if (rc) return rc;
    }
  } else {
    if (!y || ldy < N || ldy % 8 || (reinterpret_cast<uintptr_t>(y) & 15)) {
      autosp_set_error("qkv_gemm: local output needs a 16-byte aligned Y with ldy >= N");
      return AUTOSP_ERR_VALIDATION;
    }
    p.y = static_cast<__nv_bfloat16*>(y);
    p.ldy = ldy;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int tiles = (M / BM) * (N / BN);
  const int grid = tiles < sms ? tiles : sms;
  static bool attr[3] = {false, false, false};
  cudaError_t e = cudaSuccess;
  switch (d) {
    case 32:
      if (!attr[0]) cudaFuncSetAttribute(qkv_gemm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM), attr[0] = true;
      qkv_gemm_kernel<32><<<grid, kThreads, SMEM, st>>>(p);
      break;
    case 64:
      if (!attr[1]) cudaFuncSetAttribute(qkv_gemm_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM), attr[1] = true;
      qkv_gemm_kernel<64><<<grid, kThreads, SMEM, st>>>(p);
      break;
    default:
      if (!attr[2]) cudaFuncSetAttribute(qkv_gemm_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM), attr[2] = true;
      qkv_gemm_kernel<128><<<grid, kThreads, SMEM, st>>>(p);
      break;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    autosp_set_error("qkv_gemm launch failed: %s", cudaGetErrorString(e));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}

int autosp_preload_gemm() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, autosp::gemm::qkv_gemm_kernel<32>);
  cudaFuncGetAttributes(&a, autosp::gemm::qkv_gemm_kernel<64>);
  cudaFuncGetAttributes(&a, autosp::gemm::qkv_gemm_kernel<128>);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
