// K4: causal flash-attention backward for the local head block (the gradient of the
// AttentionCore, reference recipes autodiff.py:156-162 (batch-matmul grads),
// autodiff.py:190-195 (scale), autodiff.py:213-214 + executor.py:89-91 (softmax_dx)),
// recomputing P from the forward's LSE instead of saving the O(s^2) probabilities.
//
// Three launches, all stream-ordered:
//   bwd_pre   delta = rowsum(dO * O) (fp32), zero the fp32 dQ accumulator
//   bwd_main  one CTA per (batch, kv head, 128-key tile); loops over every q head of the
//             GQA group and every query tile at/after the diagonal:
//               S^T  = K Q^T        (tcgen05, SS)       -> TMEM
//               dP^T = V dO^T       (tcgen05, SS)       -> TMEM
//               P^T  = exp2(S^T*c - lse), dS^T = P^T (dP^T - delta)   (softmax warps,
//                      thread = key row; bf16 P^T/dS^T written back to TMEM, dS^T also to
//                      a 128B-swizzled smem tile)
//               dV  += P^T dO       (TS: A from TMEM)
//               dK  += dS^T Q       (TS)
//               dQ_t = dS K         (SS, A = dS^T smem read MN-major) -> TMEM, drained by
//                      a second warpgroup into smem and TMA-reduce-added (fp32) into dQacc
//             dK/dV stay in TMEM for the whole CTA (GQA reduction is free) and are written
//             once at the end.
//   bwd_post  dq = bf16(scale * dQacc)
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/autosp.h"
#include "ptx.cuh"
#include "tma.cuh"

extern "C" void autosp_set_error(const char* fmt, ...);
int autosp_check_attn_tensor(const autosp_attn_tensor& t, const char* name);

namespace autosp {
namespace bwd {

constexpr int BK = 128;  // keys per CTA
constexpr int BQ = 128;  // queries per step
constexpr int kThreads = 384;

AUTOSP_DEV void tma_reduce_add_3d(const CUtensorMap* map, const void* smem, int c0, int c1,
                                  int c2) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, "
      "%4}], [%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
AUTOSP_DEV void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}

template <int D>
struct Cfg {
  static constexpr int SW = (D * 2 >= 128) ? 128 : D * 2;
  static constexpr int CE = SW / 2;
  static constexpr int NCH = D / CE;
  static constexpr int LAYOUT = SW == 128 ? 2 : (SW == 64 ? 4 : 6);
  static constexpr int SBO = 8 * SW;
  static constexpr int TILE = 128 * D * 2;  // one [128 x D] bf16 tile
  static constexpr int kQStages = D == 128 ? 1 : 2;
  // S^T buffers in TMEM: two (S(t+1) overlaps the softmax of t) when d <= 64
  static constexpr int NSB = D == 128 ? 1 : 2;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = TILE;
  static constexpr int Q_OFF = 2 * TILE;                       // Q[st]
  static constexpr int DO_OFF = Q_OFF + kQStages * TILE;       // dO[st]
  static constexpr int DS_OFF = DO_OFF + kQStages * TILE;      // dS^T [128 keys x 128 q] bf16
  static constexpr int DQ_OFF = DS_OFF + 128 * 128 * 2;        // 2 fp32 chunks [128 x 32]
  static constexpr int LSE_OFF = DQ_OFF + 2 * 128 * 32 * 4;    // lse[st][128], delta[st][128]
  static constexpr int BAR_OFF = LSE_OFF + 4 * 128 * 4;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  // TMEM columns.  d <= 64: S0 | S1 | dP (dS bf16 in cols 0..63, dQ fp32 in 64..64+D) | dV | dK
  //                d = 128: S (dQ reuses it after dV consumed P) | dP | dV | dK
  static constexpr uint32_t DP_COL = NSB * 128;
  static constexpr uint32_t DV_COL = DP_COL + 128;
  static constexpr uint32_t DK_COL = DV_COL + D;
  static constexpr uint32_t DQ_COL = NSB == 2 ? DP_COL + 64 : 0;
  static_assert(DK_COL + D <= 512, "TMEM budget");
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v, tm_do, tm_dqacc, tm_lse, tm_dlt;
  int lse_tma;         // lse/delta rows staged by TMA with Q/dO (needs S % 4 == 0)
  const float* lse;    // [B, Hq, S]
  const float* delta;  // [B, Hq, S]
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  int64_t dk_sb, dk_sh, dk_ss, dv_sb, dv_sh, dv_ss;
  int B, Hq, Hkv, S;
  float scale, scale_log2;
  int causal;
  int n_ktiles;
};

template <int D>
AUTOSP_DEV uint64_t desc_kmajor(uint32_t tile_saddr, int kk) {
  using C = Cfg<D>;
  const int e = kk * 16;
  return make_smem_desc(tile_saddr + (e / C::CE) * (128 * C::SW) + (e % C::CE) * 2, 16, C::SBO,
                        C::LAYOUT);
}
// MN-major operand stored as [128 K-rows x D] in NCH chunks: step kk covers 16 K-rows.
template <int D>
AUTOSP_DEV uint64_t desc_mn(uint32_t tile_saddr, int kk) {
  using C = Cfg<D>;
  return make_smem_desc(tile_saddr + kk * 16 * C::SW, 128 * C::SW, C::SBO, C::LAYOUT);
}
// dS^T smem tile [128 keys x 128 queries] bf16, two 128B-swizzled chunks of 64 queries:
// as the A operand of dQ = dS K it is MN-major (M = queries contiguous), K = keys.
AUTOSP_DEV uint64_t desc_ds(uint32_t saddr, int kk) {
  return make_smem_desc(saddr + kk * 16 * 128, 128 * 128, 1024, 2);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;                  // [kQStages]
  uint64_t* q_empty = q_full + C::kQStages;     // [kQStages]
  uint64_t* s_full = q_empty + C::kQStages;     // [NSB] S^T(t) in TMEM
  uint64_t* dp_full = s_full + 2;               // dP^T(t) in TMEM
  uint64_t* p_ready = dp_full + 1;              // P^T written (128 arrivals)
  uint64_t* ds_ready = p_ready + 1;             // dS^T written to TMEM + smem (128 arrivals)
  uint64_t* dq_full = ds_ready + 1;             // dQ MMA complete
  uint64_t* dq_empty = dq_full + 1;             // dQ drained from TMEM (128 arrivals)
  uint64_t* acc_full = dq_empty + 1;            // final dK/dV complete
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_full + 1);
  float* lse_s = reinterpret_cast<float*>(smem + C::LSE_OFF);  // [kQStages][128]
  float* dlt_s = lse_s + 256;                                   // [kQStages][128]

  const int warp = warp_id();
  const int lane = lane_id();
  const int ktile = blockIdx.x;  // launch order = heaviest (most query tiles) first
  const int kvh = blockIdx.y;
  const int batch = blockIdx.z;
  const int group = p.Hq / p.Hkv;
  const int k0 = ktile * BK;
  const int n_qtiles = (p.S + BQ - 1) / BQ;
  const int m_first = p.causal ? (k0 / BQ) : 0;
  const int per_head = n_qtiles - m_first;
  const int T = per_head * group;  // steps of this CTA

  if (warp == 0 && lane == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < C::kQStages; ++s) {
      mbar_init(q_full + s, 1);
      mbar_init(q_empty + s, 1);
    }
    mbar_init(s_full + 0, 1);
    mbar_init(s_full + 1, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_ready, 128);
    mbar_init(ds_ready, 128);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 128);
    mbar_init(acc_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&p.tm_q);
    tma_prefetch_desc(&p.tm_k);
    tma_prefetch_desc(&p.tm_v);
    tma_prefetch_desc(&p.tm_do);
    tma_prefetch_desc(&p.tm_dqacc);
    if (p.lse_tma) {
      tma_prefetch_desc(&p.tm_lse);
      tma_prefetch_desc(&p.tm_dlt);
    }
  }
  if (warp == 2) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t s_k = smem_u32(smem + C::K_OFF);
  const uint32_t s_v = smem_u32(smem + C::V_OFF);
  const uint32_t s_q = smem_u32(smem + C::Q_OFF);
  const uint32_t s_do = smem_u32(smem + C::DO_OFF);
  const uint32_t s_ds = smem_u32(smem + C::DS_OFF);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && T > 0) {
      const uint64_t pol_last = policy_evict_last();
      mbar_arrive_expect_tx(kv_full, 2 * C::TILE);
      for (int c = 0; c < C::NCH; ++c) {
        tma_load_4d(smem + C::K_OFF + c * 128 * C::SW, &p.tm_k, kv_full, c * C::CE, k0, kvh,
                    batch, pol_last);
        tma_load_4d(smem + C::V_OFF + c * 128 * C::SW, &p.tm_v, kv_full, c * C::CE, k0, kvh,
                    batch, pol_last);
      }
      for (int t = 0; t < T; ++t) {
        const int st = t % C::kQStages;
        const uint32_t ph = (t / C::kQStages) & 1;
        const int head = kvh * group + t / per_head;
        const int q0 = (m_first + t % per_head) * BQ;
        mbar_wait(q_empty + st, ph ^ 1);
        mbar_arrive_expect_tx(q_full + st, 2 * C::TILE + (p.lse_tma ? 2 * 128 * 4 : 0));
        if (p.lse_tma) {  // the softmax warps need lse/delta of these 128 queries
          tma_load_2d(lse_s + st * 128, &p.tm_lse, q_full + st, q0, batch * p.Hq + head);
          tma_load_2d(dlt_s + st * 128, &p.tm_dlt, q_full + st, q0, batch * p.Hq + head);
        }
        for (int c = 0; c < C::NCH; ++c) {
          tma_load_4d(smem + C::Q_OFF + st * C::TILE + c * 128 * C::SW, &p.tm_q, q_full + st,
                      c * C::CE, q0, head, batch, pol_last);
          tma_load_4d(smem + C::DO_OFF + st * C::TILE + c * 128 * C::SW, &p.tm_do, q_full + st,
                      c * C::CE, q0, head, batch, pol_last);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && T > 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);   // K-major x K-major
      constexpr uint32_t idesc_g = make_idesc_bf16(128, D, 0, 1);     // TMEM A x MN-major B
      constexpr uint32_t idesc_q = make_idesc_bf16(128, D, 1, 1);     // MN-major A and B
      auto issue_s = [&](int t) {  // S^T(t) = K Q(t)^T
        const uint32_t qa = s_q + (t % C::kQStages) * C::TILE;
        mbar_wait(q_full + (t % C::kQStages), (t / C::kQStages) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + (t % C::NSB) * 128, desc_kmajor<D>(s_k, kk), desc_kmajor<D>(qa, kk),
                 idesc_s, kk > 0);
        tc_commit(s_full + (t % C::NSB));
      };
      mbar_wait(kv_full, 0);
      if (C::NSB == 2) issue_s(0);
      for (int t = 0; t < T; ++t) {
        const int st = t % C::kQStages;
        const uint32_t qa = s_q + st * C::TILE;
        const uint32_t da = s_do + st * C::TILE;
        const uint32_t s_col = (t % C::NSB) * 128;
        // the dP region (and for d = 128 the S region) held dQ(t-1): wait for its drain
        if (t > 0) {
          mbar_wait(dq_empty, (t - 1) & 1);
          tc_fence_after();
        }
        if (C::NSB == 1) issue_s(t);
        else {
          mbar_wait(q_full + st, (t / C::kQStages) & 1);
          tc_fence_after();
        }
        // dP^T(t) = V dO(t)^T
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem + C::DP_COL, desc_kmajor<D>(s_v, kk), desc_kmajor<D>(da, kk), idesc_s,
                 kk > 0);
        tc_commit(dp_full);
        // S^T(t+1) overlaps the softmax of tile t (its buffer held P(t-1): consumed by
        // dV(t-1), issued earlier -> in-order)
        if (C::NSB == 2 && t + 1 < T) issue_s(t + 1);
        // dV += P^T dO once the exps of tile t are done
        mbar_wait(p_ready, t & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk)
          mma_ts(tmem + C::DV_COL, tmem + s_col + kk * 8, desc_mn<D>(da, kk), idesc_g,
                 (t > 0 || kk > 0) ? 1u : 0u);
        // dK += dS^T Q and dQ(t) = dS K once dS is in TMEM + smem
        mbar_wait(ds_ready, t & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk)
          mma_ts(tmem + C::DK_COL, tmem + C::DP_COL + kk * 8, desc_mn<D>(qa, kk), idesc_g,
                 (t > 0 || kk > 0) ? 1u : 0u);
        tc_commit(q_empty + st);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          mma_ss(tmem + C::DQ_COL, desc_ds(s_ds, kk), desc_mn<D>(s_k, kk), idesc_q, kk > 0);
        tc_commit(dq_full);
      }
      tc_commit(acc_full);
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ softmax-grad warpgroup
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // key row within the tile
    const int key = k0 + row;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t dp_addr = tmem + lane_base + C::DP_COL;
    uint8_t* ds_row = smem + C::DS_OFF + row * 128;
    const float LOG2E = 1.4426950408889634f;
    for (int t = 0; t < T; ++t) {
      const int head = kvh * group + t / per_head;
      const int q0 = (m_first + t % per_head) * BQ;
      const uint32_t s_addr = tmem + lane_base + (t % C::NSB) * 128;
      const int st = t % C::kQStages;
      float* lse_b = lse_s + st * 128;
      float* dlt_b = dlt_s + st * 128;
      if (!p.lse_tma) {  // S % 4 != 0: stage lse/delta through registers (slow path)
        if (t >= C::kQStages) named_bar_sync(1, 128);  // everyone done with this slot
        const int q = q0 + row;
        const int64_t idx = ((int64_t)batch * p.Hq + head) * p.S + q;
        lse_b[row] = q < p.S ? p.lse[idx] : 0.f;
        dlt_b[row] = q < p.S ? p.delta[idx] : 0.f;
        named_bar_sync(1, 128);
      }
      const bool diag = p.causal && (q0 < k0 + BK);
      const bool oob = (k0 + BK > p.S) || (q0 + BQ > p.S);
      // ---- part 1: P^T = exp2(S^T c - lse) -> bf16 into the S columns
      mbar_wait(s_full + (t % C::NSB), (t / C::NSB) & 1);
      tc_fence_after();
#pragma unroll
      for (int c4 = 0; c4 < BQ / 32; ++c4) {
        uint32_t sr[32], pk[16];
        tmem_ld32(s_addr + c4 * 32, sr);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          float pv[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = c4 * 32 + 2 * c + e;
            float pp = fast_exp2(fmaf(__uint_as_float(sr[2 * c + e]), p.scale_log2,
                                      -lse_b[col] * LOG2E));
            if ((diag || oob) &&
                ((p.causal && key > q0 + col) || key >= p.S || q0 + col >= p.S))
              pp = 0.f;
            pv[e] = pp;
          }
          pk[c] = pack_bf16(pv[0], pv[1]);
        }
        tmem_st16(s_addr + c4 * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_ready);
      // ---- part 2: dS^T = P^T (dP^T - delta) -> bf16 into the dP columns and smem
      // (dp_full(t) also implies dQ(t-1) finished reading the smem dS tile)
      mbar_wait(dp_full, t & 1);
      tc_fence_after();
#pragma unroll
      for (int c4 = 0; c4 < BQ / 32; ++c4) {
        uint32_t dr[32], pk[16];
        tmem_ld32(dp_addr + c4 * 32, dr);
        tmem_ld16(s_addr + c4 * 16, pk);  // P^T (bf16) written in part 1
        tmem_wait_ld();
        uint32_t dk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int col = c4 * 32 + 2 * c;
          const float2 pf = __bfloat1622float2(
              *reinterpret_cast<const __nv_bfloat162*>(&pk[c]));
          float d0 = dlt_b[col], d1 = dlt_b[col + 1];
          if (oob) {  // TMA zero-fills rows past S; keep 0 * (x - garbage) out of dS
            d0 = (q0 + col < p.S) ? d0 : 0.f;
            d1 = (q0 + col + 1 < p.S) ? d1 : 0.f;
          }
          dk[c] = pack_bf16(pf.x * (__uint_as_float(dr[2 * c]) - d0),
                            pf.y * (__uint_as_float(dr[2 * c + 1]) - d1));
        }
        tmem_st16(dp_addr + c4 * 16, dk);
        uint8_t* chunk = ds_row + (c4 >> 1) * (128 * 128);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int unit = (c4 & 1) * 4 + u;  // 16-byte unit within the 128 B row
          *reinterpret_cast<uint4*>(chunk + ((unit ^ (row & 7)) << 4)) =
              make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
        }
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(ds_ready);
    }
    // ---- epilogue: dV, dK (scaled) straight from TMEM
    if (T > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
      const uint32_t dv_addr = tmem + lane_base + C::DV_COL;
      const uint32_t dk_addr = tmem + lane_base + C::DK_COL;
      __nv_bfloat16* dvrow = p.dv + (int64_t)batch * p.dv_sb + (int64_t)kvh * p.dv_sh +
                             (int64_t)key * p.dv_ss;
      __nv_bfloat16* dkrow = p.dk + (int64_t)batch * p.dk_sb + (int64_t)kvh * p.dk_sh +
                             (int64_t)key * p.dk_ss;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t a[32], g[32];
        tmem_ld32(dv_addr + c, a);
        tmem_ld32(dk_addr + c, g);
        tmem_wait_ld();
        if (key < p.S) {
#pragma unroll
          for (int t4 = 0; t4 < 4; ++t4) {
            uint4 va, vg;
            va.x = pack_bf16(__uint_as_float(a[8 * t4 + 0]), __uint_as_float(a[8 * t4 + 1]));
            va.y = pack_bf16(__uint_as_float(a[8 * t4 + 2]), __uint_as_float(a[8 * t4 + 3]));
            va.z = pack_bf16(__uint_as_float(a[8 * t4 + 4]), __uint_as_float(a[8 * t4 + 5]));
            va.w = pack_bf16(__uint_as_float(a[8 * t4 + 6]), __uint_as_float(a[8 * t4 + 7]));
            vg.x = pack_bf16(__uint_as_float(g[8 * t4 + 0]) * p.scale,
                             __uint_as_float(g[8 * t4 + 1]) * p.scale);
            vg.y = pack_bf16(__uint_as_float(g[8 * t4 + 2]) * p.scale,
                             __uint_as_float(g[8 * t4 + 3]) * p.scale);
            vg.z = pack_bf16(__uint_as_float(g[8 * t4 + 4]) * p.scale,
                             __uint_as_float(g[8 * t4 + 5]) * p.scale);
            vg.w = pack_bf16(__uint_as_float(g[8 * t4 + 6]) * p.scale,
                             __uint_as_float(g[8 * t4 + 7]) * p.scale);
            reinterpret_cast<uint4*>(dvrow + c)[t4] = va;
            reinterpret_cast<uint4*>(dkrow + c)[t4] = vg;
          }
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ dQ drain warpgroup
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // query row within the step
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t dq_addr = tmem + lane_base + C::DQ_COL;
    const bool leader = (warp == 8 && lane == 0);
    for (int t = 0; t < T; ++t) {
      const int head = kvh * group + t / per_head;
      const int q0 = (m_first + t % per_head) * BQ;
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float* slot = reinterpret_cast<float*>(smem + C::DQ_OFF) + (c & 1) * (128 * 32);
        if (leader) bulk_wait_read1();  // the reduce that last used this slot has read it
        named_bar_sync(2, 128);
        uint32_t v[32];
        tmem_ld32(dq_addr + c * 32, v);
        tmem_wait_ld();
        uint8_t* srow = reinterpret_cast<uint8_t*>(slot) + row * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<uint4*>(srow + ((u ^ (row & 7)) << 4)) =
              make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
        fence_proxy_async_smem();
        named_bar_sync(2, 128);
        if (leader) {
          tma_reduce_add_3d(&p.tm_dqacc, slot, c * 32, q0, batch * p.Hq + head);
          bulk_commit();
        }
      }
      tc_fence_before();
      mbar_arrive(dq_empty);
    }
    if (leader) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------- pre / post
struct PrePost {
  const __nv_bfloat16* o;
  const __nv_bfloat16* d_o;
  __nv_bfloat16* dq;
  int64_t o_sb, o_sh, o_ss, do_sb, do_sh, do_ss, dq_sb, dq_sh, dq_ss;
  float* dqacc;
  float* delta;
  int Hq, S, D;
  int64_t rows;
  float scale;
};

// delta[row] = sum_d dO*O ; dqacc[row, :] = 0.  lanes_per_row = D/8 (one 16B vector each).
__global__ void bwd_pre_kernel(const __grid_constant__ PrePost a) {
  const int lpr = a.D / 8;
  const int rpw = 32 / lpr;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t row = warp * rpw + lane / lpr;
  const int sub = lane % lpr;
  float acc = 0.f;
  if (row < a.rows) {
    const int64_t bh = row / a.S;
    const int q = (int)(row % a.S);
    const int h = (int)(bh % a.Hq);
    const int64_t bi = bh / a.Hq;
    const uint4 ov = *reinterpret_cast<const uint4*>(a.o + bi * a.o_sb + h * a.o_sh +
                                                     (int64_t)q * a.o_ss + sub * 8);
    const uint4 gv = *reinterpret_cast<const uint4*>(a.d_o + bi * a.do_sb + h * a.do_sh +
                                                     (int64_t)q * a.do_ss + sub * 8);
    const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __bfloat1622float2(o2[i]);
      const float2 y = __bfloat1622float2(g2[i]);
      acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
    }
    float4* z = reinterpret_cast<float4*>(a.dqacc + row * a.D + sub * 8);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int off = lpr / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (row < a.rows && sub == 0) a.delta[row] = acc;
}

__global__ void bwd_post_kernel(const __grid_constant__ PrePost a) {
  const int lpr = a.D / 8;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid / lpr;
  const int sub = (int)(gid % lpr);
  if (row >= a.rows) return;
  const int64_t bh = row / a.S;
  const int q = (int)(row % a.S);
  const int h = (int)(bh % a.Hq);
  const int64_t bi = bh / a.Hq;
  const float4* src = reinterpret_cast<const float4*>(a.dqacc + row * a.D + sub * 8);
  const float4 x = src[0], y = src[1];
  uint4 v;
  v.x = pack_bf16(x.x * a.scale, x.y * a.scale);
  v.y = pack_bf16(x.z * a.scale, x.w * a.scale);
  v.z = pack_bf16(y.x * a.scale, y.y * a.scale);
  v.w = pack_bf16(y.z * a.scale, y.w * a.scale);
  *reinterpret_cast<uint4*>(a.dq + bi * a.dq_sb + h * a.dq_sh + (int64_t)q * a.dq_ss + sub * 8) =
      v;
}

inline bool make_map_f32_3d(CUtensorMap* map, void* ptr, int BH, int S, int D) {
  PFN_encodeTiled enc = get_encode_tiled();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)S, (cuuint64_t)BH};
  cuuint64_t strides[2] = {(cuuint64_t)D * 4, (cuuint64_t)S * D * 4};
  cuuint32_t box[3] = {32, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// [rows, S] fp32 (row stride S), box {128, 1}: one query tile of lse / delta
inline bool make_map_rows_f32(CUtensorMap* map, const void* ptr, int rows, int S) {
  PFN_encodeTiled enc = get_encode_tiled();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)S, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)S * 4};
  cuuint32_t box[2] = {128, 1};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <int D>
int launch(const autosp_attn_tensor& q, const autosp_attn_tensor& k, const autosp_attn_tensor& v,
           const autosp_attn_tensor& o, const autosp_attn_tensor& d_o, const float* lse,
           const autosp_attn_tensor& dq, const autosp_attn_tensor& dk,
           const autosp_attn_tensor& dv, void* ws, int B, int Hq, int Hkv, int S, float scale,
           int causal, cudaStream_t stream) {
  using C = Cfg<D>;
  float* dqacc = static_cast<float*>(ws);
  float* delta = dqacc + (size_t)B * Hq * S * D;
  PrePost a{};
  a.o = static_cast<const __nv_bfloat16*>(o.ptr);
  a.d_o = static_cast<const __nv_bfloat16*>(d_o.ptr);
  a.dq = static_cast<__nv_bfloat16*>(const_cast<void*>(dq.ptr));
  a.o_sb = o.stride_b; a.o_sh = o.stride_h; a.o_ss = o.stride_s;
  a.do_sb = d_o.stride_b; a.do_sh = d_o.stride_h; a.do_ss = d_o.stride_s;
  a.dq_sb = dq.stride_b; a.dq_sh = dq.stride_h; a.dq_ss = dq.stride_s;
  a.dqacc = dqacc;
  a.delta = delta;
  a.Hq = Hq;
  a.S = S;
  a.D = D;
  a.rows = (int64_t)B * Hq * S;
  a.scale = scale;
  {
    const int rpw = 32 / (D / 8);
    const int64_t warps = (a.rows + rpw - 1) / rpw;
    const int64_t blocks = (warps * 32 + 255) / 256;
    bwd_pre_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a);
  }
  Params p{};
  bool ok = make_map_bhsd(&p.tm_q, q.ptr, B, Hq, S, D, q.stride_b, q.stride_h, q.stride_s, C::CE,
                          128, C::SW) &&
            make_map_bhsd(&p.tm_do, d_o.ptr, B, Hq, S, D, d_o.stride_b, d_o.stride_h,
                          d_o.stride_s, C::CE, 128, C::SW) &&
            make_map_bhsd(&p.tm_k, k.ptr, B, Hkv, S, D, k.stride_b, k.stride_h, k.stride_s,
                          C::CE, 128, C::SW) &&
            make_map_bhsd(&p.tm_v, v.ptr, B, Hkv, S, D, v.stride_b, v.stride_h, v.stride_s,
                          C::CE, 128, C::SW) &&
            make_map_f32_3d(&p.tm_dqacc, dqacc, B * Hq, S, D);
  p.lse_tma = (S % 4 == 0) && make_map_rows_f32(&p.tm_lse, lse, B * Hq, S) &&
              make_map_rows_f32(&p.tm_dlt, delta, B * Hq, S);
  if (!ok) {
    autosp_set_error("attn_bwd: cuTensorMapEncodeTiled failed (alignment/strides?)");
    return AUTOSP_ERR_VALIDATION;
  }
  p.lse = lse;
  p.delta = delta;
  p.dk = static_cast<__nv_bfloat16*>(const_cast<void*>(dk.ptr));
  p.dv = static_cast<__nv_bfloat16*>(const_cast<void*>(dv.ptr));
  p.dk_sb = dk.stride_b; p.dk_sh = dk.stride_h; p.dk_ss = dk.stride_s;
  p.dv_sb = dv.stride_b; p.dv_sh = dv.stride_h; p.dv_ss = dv.stride_s;
  p.B = B;
  p.Hq = Hq;
  p.Hkv = Hkv;
  p.S = S;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.causal = causal;
  p.n_ktiles = (S + BK - 1) / BK;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr_set = true;
  }
  attn_bwd_kernel<D><<<dim3(p.n_ktiles, Hkv, B), kThreads, C::SMEM, stream>>>(p);
  {
    const int64_t threads = a.rows * (D / 8);
    bwd_post_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    autosp_set_error("attn_bwd launch failed: %s", cudaGetErrorString(e));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}

}  // namespace bwd
}  // namespace autosp

extern "C" size_t autosp_attn_bwd_workspace_bytes(int b, int hq, int s, int d) {
  return (size_t)b * hq * s * (d + 1) * sizeof(float);
}

extern "C" int autosp_attn_bwd(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                               autosp_attn_tensor o, autosp_attn_tensor d_o, const float* lse,
                               autosp_attn_tensor dq, autosp_attn_tensor dk,
                               autosp_attn_tensor dv, void* workspace, int b, int hq, int hkv,
                               int s, int d, float scale, int causal, void* stream) {
  if (b < 1 || hq < 1 || hkv < 1 || s < 1 || hq % hkv) {
    autosp_set_error("attn_bwd: bad shape b=%d hq=%d hkv=%d s=%d", b, hq, hkv, s);
    return AUTOSP_ERR_VALIDATION;
  }
  int rc;
  if ((rc = autosp_check_attn_tensor(q, "q")) || (rc = autosp_check_attn_tensor(k, "k")) ||
      (rc = autosp_check_attn_tensor(v, "v")) || (rc = autosp_check_attn_tensor(o, "o")) ||
      (rc = autosp_check_attn_tensor(d_o, "do")) || (rc = autosp_check_attn_tensor(dq, "dq")) ||
      (rc = autosp_check_attn_tensor(dk, "dk")) || (rc = autosp_check_attn_tensor(dv, "dv")))
    return rc;
  if (!lse || !workspace || (reinterpret_cast<uintptr_t>(workspace) & 127)) {
    autosp_set_error("attn_bwd: lse/workspace must be non-null, workspace 128B aligned");
    return AUTOSP_ERR_VALIDATION;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (d) {
    case 32:
      return autosp::bwd::launch<32>(q, k, v, o, d_o, lse, dq, dk, dv, workspace, b, hq, hkv, s,
                                     scale, causal, st);
    case 64:
      return autosp::bwd::launch<64>(q, k, v, o, d_o, lse, dq, dk, dv, workspace, b, hq, hkv, s,
                                     scale, causal, st);
    case 128:
      return autosp::bwd::launch<128>(q, k, v, o, d_o, lse, dq, dk, dv, workspace, b, hq, hkv, s,
                                      scale, causal, st);
    default:
      autosp_set_error("attn_bwd: head_dim %d unsupported (32, 64, 128)", d);
      return AUTOSP_ERR_UNSUPPORTED;
  }
}
