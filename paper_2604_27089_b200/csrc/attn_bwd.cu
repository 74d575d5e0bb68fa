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
#include <cstdlib>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "../../include/autosp.h"
#include "flags.cuh"
#include "ptx.cuh"
#include "tma.cuh"

extern "C" void autosp_set_error(const char* fmt, ...);
int autosp_check_attn_tensor(const autosp_attn_tensor& t, const char* name);

#ifndef AUTOSP_BWD_LPT
#define AUTOSP_BWD_LPT 0  // LPT grid layout (ptx.cuh); A/B: -3 % at the bench shape (L2 sharing
#endif                    // of Q / dO between co-running key tiles), mixed at per-rank shapes
#define BWD_RANK_IDX AUTOSP_BLOCK_RANK(AUTOSP_BWD_LPT)
#define BWD_HEAD_IDX AUTOSP_BLOCK_HEAD(AUTOSP_BWD_LPT)
#ifndef AUTOSP_BWD_EMU
#define AUTOSP_BWD_EMU 2  // exps per 8 on the FMA pipe for d <= 64 (tools/emu sweep)
#endif
#ifndef AUTOSP_BWD_EMU128
#define AUTOSP_BWD_EMU128 1  // exps per 8 on the FMA pipe for d = 128
#endif

#ifndef AUTOSP_BWD_ABL
#define AUTOSP_BWD_ABL 0  // timing ablations (WRONG results, tools only): 1 no dQ staging /
#endif                    // reduce, 2 no dS smem stores, 3 no exps (P = S), 4 = 1 + 2

namespace autosp {
namespace bwd {

long long* g_bwd_trace = nullptr;  // set by autosp_debug_set_bwd_trace (tools only)

constexpr int BK = 128;  // keys per CTA
constexpr int BQ = 128;  // queries per step
constexpr int kSoftWarp0 = 4;   // softmax-grad warpgroups from warp 4 on
constexpr int kDrainWarp0 = 0;  // warps 0-3 (lowest priority: the drain has a step of slack)
constexpr int kThreads = 512;
// Warp roles (the issue arbiter favours higher warp ids: the single-thread TMA / MMA
// producers sit on top, the dQ drain below the instruction-heavy softmax warpgroups).
// (Measured and removed in round 2: 4 softmax-grad warpgroups of 32 query columns -- 2 %
// slower; busy-polling mbarrier waits -- neutral.  DESIGN.md section 7.)
constexpr int kAllocWarp = 12;
constexpr int kTmaWarp = 14;
constexpr int kMmaWarp = 15;

AUTOSP_DEV void tma_reduce_add_3d(const CUtensorMap* map, const void* smem, int c0, int c1,
                                  int c2) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, "
      "%4}], [%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
template <int N>
AUTOSP_DEV void bulk_wait_read_n() {  // at most N bulk groups still reading their smem source
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int D>
struct Cfg {
  static constexpr int SW = (D * 2 >= 128) ? 128 : D * 2;
  static constexpr int CE = SW / 2;
  static constexpr int NCH = D / CE;
  static constexpr int LAYOUT = SW == 128 ? 2 : (SW == 64 ? 4 : 6);
  static constexpr int SBO = 8 * SW;
  static constexpr int TILE = 128 * D * 2;  // one [128 x D] bf16 tile
  // Q(+lse/delta) ring depth (3 measured slower than 2 for d = 64) and dO ring depth.
  // d = 128: Q is double-buffered so S^T(t+1) can be issued right after dV(t) (it only
  // needs Q(t+1)); dO stays single (freed by dV(t), needed by dP(t+1) much later).
#ifndef AUTOSP_BWD_QSTAGES64
#define AUTOSP_BWD_QSTAGES64 3
#endif
  static constexpr int kQStages = D == 128 ? 2 : AUTOSP_BWD_QSTAGES64;
  static constexpr int kDOStages = D == 128 ? 1 : 2;
  // S^T buffers in TMEM: two (S(t+1) overlaps the softmax of t) when d <= 64
  static constexpr int NSB = D == 128 ? 1 : 2;
  // exps per 8 done on the FMA pipe (part 1 is MUFU-bound at 16 exp/clk/SM)
  static constexpr int kEmuPer8 = D == 128 ? AUTOSP_BWD_EMU128 : AUTOSP_BWD_EMU;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = TILE;
  static constexpr int Q_OFF = 2 * TILE;                       // Q[st]
  static constexpr int DO_OFF = Q_OFF + kQStages * TILE;       // dO[st]
  static constexpr int DS_OFF = DO_OFF + kDOStages * TILE;     // dS^T [128 keys x 128 q] bf16
  // dQ staging slots (fp32 [128 x 32] chunks) between the drain and the TMA reduce-add
#ifndef AUTOSP_BWD_DQSLOTS64
#define AUTOSP_BWD_DQSLOTS64 2
#endif
  static constexpr int DQS = D <= 64 ? AUTOSP_BWD_DQSLOTS64 : 2;
  static constexpr int DQ_OFF = DS_OFF + 128 * 128 * 2;
  static constexpr int LSE_OFF = DQ_OFF + DQS * 128 * 32 * 4;  // lse[kQStages][128], delta[kQStages][128]
  static constexpr int BAR_OFF = LSE_OFF + 2 * kQStages * 128 * 4;
  // dynamic smem starts 1024-aligned when the kernel has no static smem (measured:
  // shared address 0x400, tools/microbench/smem_align); d = 128 needs the slack bytes
  static constexpr int kAlignSlack = D == 128 ? 0 : 1024;
  static constexpr int SMEM = BAR_OFF + 256 + kAlignSlack;
  static_assert(SMEM <= 232448, "shared memory budget (227 KB)");
  // TMEM columns.  d <= 64: S0 | S1 | dP | dV | dK; P^T(t) (bf16) occupies columns
  //   [0,32) and [96,128) of S buffer t%2 and dQ(t) (fp32) columns [32, 32+d), so dP(t+1)
  //   never waits for the dQ drain (only S(t+2) does).
  // d = 128: S | dP | dV | dK; dQ(t) lands in the dP columns after dK(t) consumed dS(t),
  //   so S(t+1) (and the exps of t+1) overlap the dQ drain; dP(t+1) waits for it.
  static constexpr uint32_t DP_COL = NSB * 128;
  static constexpr uint32_t DV_COL = DP_COL + 128;
  static constexpr uint32_t DK_COL = DV_COL + D;
  static_assert(DK_COL + D <= 512, "TMEM budget");
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v, tm_do, tm_dqacc, tm_lse, tm_dlt;
  int lse_tma;         // lse/delta rows staged by TMA with Q/dO (needs S % 4 == 0)
  long long* trace;    // debug timeline (nullptr in production): [16 events][kTraceSteps]
  float* dqacc;        // [B, Hq, S, D] fp32 accumulator (red.global.add from the drain)
  const float* lse;    // [B, Hq, S]  -lse * log2(e) (written by bwd_pre)
  const float* delta;  // [B, Hq, S]
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  int64_t dk_sb, dk_sh, dk_ss, dv_sb, dv_sh, dv_ss;
  int B, Hq, Hkv, S;
  float scale, scale_log2;
  int causal;
  int n_ktiles;
  // fused head->seq all-to-all of the gradients (autosp_attn_bwd_push): dK / dV rows go
  // straight into the token owner's packed [b, s/P, hq+2hkv, d] QKV gradient (global
  // heads hq*P + rank*hkv + kvh and hq*P + hkv*P + rank*hkv + kvh); push == 0: local
  int push, P, rank, s_loc;
  int64_t dst_off, d_sb, d_ss, d_sh;  // bytes / elements
  char* peer_base[AUTOSP_MAX_WORLD];
  // GQA split (small grids, e.g. one kv head per rank at SP = 8): hsplit CTAs share a
  // (key tile, kv head), each taking group/hsplit of its q heads; their dK/dV partials are
  // red.add-ed into dkv_acc (fp32 [2][B][Hkv][S][D]: dK, dV) and bwd_post finishes them.
  // With hsplit = 2 every element gets exactly two addends: deterministic.
  int hsplit;
  float* dkv_acc;
};

constexpr int kTraceSteps = 64;
#define BWD_TRACE(ev, t)                                                                  \
  do {                                                                                    \
    if (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (t) < kTraceSteps) \
      p.trace[(ev) * kTraceSteps + (t)] = clock64();                                      \
  } while (0)

template <int D>
AUTOSP_DEV uint64_t desc_kmajor(uint32_t tile_saddr, int kk) {
  using C = Cfg<D>;
  const int e = kk * 16;
  return make_smem_desc(tile_saddr + (e / C::CE) * (128 * C::SW) + (e % C::CE) * 2, 16, C::SBO,
                        C::LAYOUT);
}
template <int D>
__host__ __device__ constexpr uint64_t kmajor_off(int kk) {  // (byte offset of K-step kk) >> 4
  return (uint64_t)((((kk * 16) / Cfg<D>::CE) * (128 * Cfg<D>::SW) + ((kk * 16) % Cfg<D>::CE) * 2) >> 4);
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

// PUSH (compile-time): the fused head->seq push of dK/dV (autosp_attn_bwd_push); a separate
// instantiation keeps the local-output kernel free of the push path's register pressure
template <int D, bool PUSH, bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;                  // [kQStages]
  uint64_t* q_empty = q_full + C::kQStages;     // [kQStages]
  uint64_t* s_full = q_empty + C::kQStages;     // [2] S^T(t) in TMEM
  uint64_t* dp_full = s_full + 2;               // dP^T(t) in TMEM
  uint64_t* p_ready = dp_full + 1;              // P^T written (256 arrivals)
  uint64_t* ds_ready = p_ready + 1;             // dS^T written to TMEM + smem (256 arrivals)
  uint64_t* dq_full = ds_ready + 1;             // dQ MMA complete
  uint64_t* dq_empty = dq_full + 1;             // dQ drained from TMEM (128 arrivals)
  uint64_t* acc_full = dq_empty + 1;            // final dK/dV complete
  uint64_t* do_full = acc_full + 1;             // [kDOStages] dO(t) in smem
  uint64_t* do_empty = do_full + C::kDOStages;  // [kDOStages] dP(t), dV(t) done with it
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(do_empty + C::kDOStages);
  float* lse_s = reinterpret_cast<float*>(smem + C::LSE_OFF);  // [kQStages][128]
  float* dlt_s = lse_s + C::kQStages * 128;                                   // [kQStages][128]

  if constexpr (C::kAlignSlack == 0) {
    if (smem_u32(smem_raw) & 1023) asm volatile("trap;");  // layout assumes 1024 alignment
  }
  const int warp = warp_id();
  const int lane = lane_id();
  const int ktile = BWD_RANK_IDX;  // launch order = heaviest (most query tiles) first
  constexpr int HS = SPLIT ? 2 : 1;                            // (compile-time: registers)
  const int kvh = BWD_HEAD_IDX / HS;
  const int batch = blockIdx.z;
  const int group = p.Hq / p.Hkv;
  const int gsz = group / HS;                                  // q heads of this CTA
  const int k0 = ktile * BK;
  const int n_qtiles = (p.S + BQ - 1) / BQ;
  const int m_first = p.causal ? (k0 / BQ) : 0;
  const int per_head = n_qtiles - m_first;
  const int T = per_head * gsz;  // steps of this CTA

  if (warp == kTmaWarp && lane == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < C::kQStages; ++s) {
      mbar_init(q_full + s, 1);
      mbar_init(q_empty + s, 1);
    }
    mbar_init(s_full + 0, 1);
    mbar_init(s_full + 1, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_ready, 8);     // one arrival per softmax warp
    mbar_init(ds_ready, 8);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 4);
    mbar_init(acc_full, 1);
    for (int s = 0; s < C::kDOStages; ++s) {
      mbar_init(do_full + s, 1);
      mbar_init(do_empty + s, 1);
    }
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
  if (warp == kAllocWarp) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t s_k = smem_u32(smem + C::K_OFF);
  const uint32_t s_v = smem_u32(smem + C::V_OFF);
  const uint32_t s_q = smem_u32(smem + C::Q_OFF);
  const uint32_t s_do = smem_u32(smem + C::DO_OFF);
  const uint32_t s_ds = smem_u32(smem + C::DS_OFF);
  // where dQ(t) accumulates (see Cfg)
  auto dq_col = [&](int t) -> uint32_t {
    return C::NSB == 2 ? (uint32_t)((t & 1) * 128 + 32) : C::DP_COL;
  };
  // bf16 P^T / dS^T of query-column half h (64 queries = 32 packed columns) are written
  // inside the columns that half itself read: h = 0 -> cols [0, 32), h = 1 -> [96, 128).
  // (Writing them densely would overwrite fp32 scores the other half may still be
  // reading.)  K-step kk (16 queries) of the TS-MMA A operand therefore lives at:
  auto pk_col = [](int kk) -> uint32_t { return kk < 4 ? kk * 8 : 96 + (kk - 4) * 8; };

  if (warp == kTmaWarp) {
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
        const int head = kvh * group + (SPLIT ? (int)(BWD_HEAD_IDX % HS) * gsz : 0) + t / per_head;
        const int q0 = (m_first + t % per_head) * BQ;
        mbar_wait(q_empty + st, ph ^ 1);
        mbar_arrive_expect_tx(q_full + st, C::TILE + (p.lse_tma ? 2 * 128 * 4 : 0));
        if (p.lse_tma) {  // the softmax warps need lse/delta of these 128 queries
          tma_load_2d(lse_s + st * 128, &p.tm_lse, q_full + st, q0, batch * p.Hq + head);
          tma_load_2d(dlt_s + st * 128, &p.tm_dlt, q_full + st, q0, batch * p.Hq + head);
        }
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(smem + C::Q_OFF + st * C::TILE + c * 128 * C::SW, &p.tm_q, q_full + st,
                      c * C::CE, q0, head, batch, pol_last);
        const int so = t % C::kDOStages;
        mbar_wait(do_empty + so, ((t / C::kDOStages) & 1) ^ 1);
        mbar_arrive_expect_tx(do_full + so, C::TILE);
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(smem + C::DO_OFF + so * C::TILE + c * 128 * C::SW, &p.tm_do, do_full + so,
                      c * C::CE, q0, head, batch, pol_last);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // Whole warp runs the schedule (uniform control flow keeps descriptors in uniform
    // registers); one elected lane issues each batch.  Descriptors are built per tile and
    // advanced by compile-time offsets.
    if (T > 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);   // K-major x K-major
      constexpr uint32_t idesc_g = make_idesc_bf16(128, D, 0, 1);     // TMEM A x MN-major B
      constexpr uint32_t idesc_q = make_idesc_bf16(128, D, 1, 1);     // MN-major A and B
      const uint64_t dk_k = make_smem_desc(s_k, 16, C::SBO, C::LAYOUT);        // K, K-major
      const uint64_t dv_k = make_smem_desc(s_v, 16, C::SBO, C::LAYOUT);        // V, K-major
      const uint64_t dk_mn = make_smem_desc(s_k, 128 * C::SW, C::SBO, C::LAYOUT);  // K, MN
      const uint64_t dds = make_smem_desc(s_ds, 128 * 128, 1024, 2);           // dS^T tile
      auto wait_q = [&](int t) {
        mbar_wait(q_full + (t % C::kQStages), (t / C::kQStages) & 1);
        tc_fence_after();
      };
      auto issue_s = [&](int t) {  // S^T(t) = K Q(t)^T into S buffer t % NSB
        const uint64_t dq = make_smem_desc(s_q + (t % C::kQStages) * C::TILE, 16, C::SBO, C::LAYOUT);
        const uint32_t d_tm = tmem + (t % C::NSB) * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_ss(d_tm, dk_k + kmajor_off<D>(kk), dq + kmajor_off<D>(kk), idesc_s, kk > 0);
          tc_commit(s_full + (t % C::NSB));
        }
        __syncwarp();
      };
      auto issue_dp = [&](int t) {  // dP^T(t) = V dO(t)^T
        mbar_wait(do_full + (t % C::kDOStages), (t / C::kDOStages) & 1);
        tc_fence_after();
        const uint64_t ddo = make_smem_desc(s_do + (t % C::kDOStages) * C::TILE, 16, C::SBO, C::LAYOUT);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_ss(tmem + C::DP_COL, dv_k + kmajor_off<D>(kk), ddo + kmajor_off<D>(kk), idesc_s,
                   kk > 0);
          tc_commit(dp_full);
        }
        __syncwarp();
      };
      mbar_wait(kv_full, 0);
      wait_q(0);
      issue_s(0);
      for (int t = 0; t < T; ++t) {
        const int st = t % C::kQStages;
        const uint64_t dq_mn = make_smem_desc(s_q + st * C::TILE, 128 * C::SW, C::SBO, C::LAYOUT);
        const uint64_t ddo_mn = make_smem_desc(s_do + (t % C::kDOStages) * C::TILE, 128 * C::SW,
                                               C::SBO, C::LAYOUT);
        const uint32_t acc0 = t > 0 ? 1u : 0u;
        if (C::NSB == 2) {
          // dP region: dS(t-1) was consumed by dK(t-1), issued earlier (in-order)
          issue_dp(t);
          if (lane == 0) BWD_TRACE(1, t);
          // S buffer (t+1)%2 holds P(t-1) (consumed by dV(t-1)) and dQ(t-1): wait drain
          // (also on the last step: every drain phase is observed before the next one)
          if (t >= 1) {
            mbar_wait(dq_empty, (t - 1) & 1);
            if (lane == 0) BWD_TRACE(0, t);
          }
          if (t + 1 < T) {
            wait_q(t + 1);
            if (lane == 0) BWD_TRACE(11, t);
            issue_s(t + 1);
            if (lane == 0) BWD_TRACE(13, t);
          }
        } else {
          // dQ(t-1) lives in the dP columns: dP(t) waits for its drain
          if (t >= 1) {
            mbar_wait(dq_empty, (t - 1) & 1);
            if (lane == 0) BWD_TRACE(0, t);
            tc_fence_after();
          }
          issue_dp(t);
          if (lane == 0) BWD_TRACE(1, t);
        }
        // dV += P^T dO once the exps of tile t are done
        mbar_wait(p_ready, t & 1);
        if (lane == 0) BWD_TRACE(2, t);
        tc_fence_after();
        const uint32_t s_col = (t % C::NSB) * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk)
            mma_ts(tmem + C::DV_COL, tmem + s_col + pk_col(kk),
                   ddo_mn + (uint64_t)((kk * 16 * C::SW) >> 4), idesc_g, kk > 0 ? 1u : acc0);
          tc_commit(do_empty + (t % C::kDOStages));  // dP(t) and dV(t) are done with dO(t)
        }
        __syncwarp();
        // d = 128: S(t+1) reuses the S columns: P(t) has been read by the softmax and is
        // consumed by dV(t), issued just above (in-order pipe).  Issuing it here instead
        // of after dK/dQ(t) lets S^T(t+1) run under the dS math of t (needs Q(t+1) only,
        // which the second Q stage has already loaded).
        if (C::NSB == 1 && t + 1 < T) {
          wait_q(t + 1);
          issue_s(t + 1);
        }
        // dK += dS^T Q and dQ(t) = dS K once dS is in TMEM + smem
        mbar_wait(ds_ready, t & 1);
        if (lane == 0) BWD_TRACE(3, t);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BQ / 16; ++kk)
            mma_ts(tmem + C::DK_COL, tmem + C::DP_COL + pk_col(kk),
                   dq_mn + (uint64_t)((kk * 16 * C::SW) >> 4), idesc_g, kk > 0 ? 1u : acc0);
          tc_commit(q_empty + st);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_ss(tmem + dq_col(t), dds + (uint64_t)((kk * 16 * 128) >> 4),
                   dk_mn + (uint64_t)((kk * 16 * C::SW) >> 4), idesc_q, kk > 0);
          tc_commit(dq_full);
        }
        __syncwarp();
        if (lane == 0) BWD_TRACE(4, t);
      }
      if (elect_one()) tc_commit(acc_full);
      __syncwarp();
      mbar_wait(dq_empty, (T - 1) & 1);  // the last drain (no phase is left unobserved)
    }
  } else if (warp >= kSoftWarp0 && warp < kSoftWarp0 + 8) {
    // ------------------------------------------------------------ softmax-grad warpgroups
    // WG1 (warps 4-7) owns query columns [0, 64), WG2 (warps 8-11) [64, 128); thread =
    // key row (TMEM lane).  Part 1: P^T = exp2(S^T c - lse log2e) -> bf16 in S columns.
    // Part 2: dS^T = P^T (dP^T - delta) -> bf16 in dP columns + 128B-swizzled smem.
    const int half = (warp - kSoftWarp0) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // key row within the tile
    const int key = k0 + row;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t dp_addr = tmem + lane_base + C::DP_COL;
    uint8_t* ds_row = smem + C::DS_OFF + half * (128 * 128) + row * 128;
    const uint64_t sl2 = f2_pack(p.scale_log2, p.scale_log2);
    const bool row_dead = key >= p.S;
    for (int t = 0; t < T; ++t) {
      const int head = kvh * group + (SPLIT ? (int)(BWD_HEAD_IDX % HS) * gsz : 0) + t / per_head;
      const int q0 = (m_first + t % per_head) * BQ;
      const uint32_t s_addr = tmem + lane_base + (t % C::NSB) * 128;
      const int st = t % C::kQStages;
      const float* lse_b = lse_s + st * 128;
      const float* dlt_b = dlt_s + st * 128;
      if (!p.lse_tma) {  // S % 4 != 0: stage lse/delta through registers (slow path)
        if (t >= C::kQStages) named_bar_sync(1, 256);  // everyone done with this slot
        if (half == 0) {
          const int q = q0 + row;
          const int64_t idx = ((int64_t)batch * p.Hq + head) * p.S + q;
          lse_s[st * 128 + row] = q < p.S ? p.lse[idx] : 0.f;
          dlt_s[st * 128 + row] = q < p.S ? p.delta[idx] : 0.f;
        }
        named_bar_sync(1, 256);
      }
      // tiles that need element masks: the diagonal (causal) and the sequence tail
      const bool masked = (p.causal && (q0 < k0 + BK)) || (k0 + BK > p.S) || (q0 + BQ > p.S);
      const int col_lo = p.causal ? key - q0 : -1;  // col < col_lo -> masked (q < key)
      const int col_hi = min(p.S - q0, BQ);          // col >= col_hi -> masked (q >= S)
      if (threadIdx.x == kSoftWarp0 * 32) BWD_TRACE(12, t);
      mbar_wait(s_full + (t % C::NSB), (t / C::NSB) & 1);
      if (threadIdx.x == kSoftWarp0 * 32) BWD_TRACE(5, t);
      tc_fence_after();
      uint32_t pkeep[32];  // this thread's 64 P^T values (bf16 pairs), reused by part 2
      auto part1 = [&](auto kMasked) {
        uint32_t sr2[2][32];  // both 32-column chunks in flight: one TMEM round trip
        tmem_ld32(s_addr + (half * 2) * 32, sr2[0]);
        tmem_ld32(s_addr + (half * 2 + 1) * 32, sr2[1]);
        tmem_wait_ld();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c4 = half * 2 + cc;  // 32-column chunk
          const uint32_t* sr = sr2[cc];
          const float4* l4 = reinterpret_cast<const float4*>(lse_b + c4 * 32);
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            const float4 l = lds128(l4 + c8);  // broadcast LDS.128
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = c8 * 2 + h;
              const uint64_t lz = h ? f2_pack(l.z, l.w) : f2_pack(l.x, l.y);
              const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(sr[2 * c]),
                                                 __uint_as_float(sr[2 * c + 1])),
                                         sl2, lz);  // lz = -lse*log2(e) (bwd_pre)
              float e0, e1;
              if (!decltype(kMasked)::value && (c & 7) >= 8 - C::kEmuPer8) {
                f2_unpack(f2_exp2_poly(x2), e0, e1);  // FMA pipe (offloads MUFU)
              } else {
                float x0, x1;
                f2_unpack(x2, x0, x1);
                e0 = AUTOSP_BWD_ABL == 3 ? x0 : fast_exp2(x0);
                e1 = AUTOSP_BWD_ABL == 3 ? x1 : fast_exp2(x1);
              }
              if constexpr (decltype(kMasked)::value) {
                const int col = c4 * 32 + 2 * c;
                e0 = (row_dead || col < col_lo || col >= col_hi) ? 0.f : e0;
                e1 = (row_dead || col + 1 < col_lo || col + 1 >= col_hi) ? 0.f : e1;
              }
              pkeep[cc * 16 + c] = pack_bf16(e0, e1);
            }
          }
          tmem_st16(s_addr + half * 96 + cc * 16,
                    *reinterpret_cast<uint32_t(*)[16]>(&pkeep[cc * 16]));
        }
      };
      if (masked) part1(std::true_type{});
      else part1(std::false_type{});
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_warp(p_ready);
      if (threadIdx.x == kSoftWarp0 * 32) BWD_TRACE(6, t);
      // (dp_full(t) also implies dQ(t-1) finished reading the smem dS tile)
      mbar_wait(dp_full, t & 1);
      if (threadIdx.x == kSoftWarp0 * 32) BWD_TRACE(7, t);
      tc_fence_after();
      auto part2 = [&](auto kMasked) {
        uint32_t dr2[2][32];
        tmem_ld32(dp_addr + (half * 2) * 32, dr2[0]);
        tmem_ld32(dp_addr + (half * 2 + 1) * 32, dr2[1]);
        tmem_wait_ld();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c4 = half * 2 + cc;
          const uint32_t* dr = dr2[cc];
          uint32_t dk[16];
          const float4* d4 = reinterpret_cast<const float4*>(dlt_b + c4 * 32);
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            float4 dl = lds128(d4 + c8);
            if constexpr (decltype(kMasked)::value) {  // rows past S (slow path garbage)
              const int col = c4 * 32 + 4 * c8;
              dl.x = col + 0 < col_hi ? dl.x : 0.f;
              dl.y = col + 1 < col_hi ? dl.y : 0.f;
              dl.z = col + 2 < col_hi ? dl.z : 0.f;
              dl.w = col + 3 < col_hi ? dl.w : 0.f;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = c8 * 2 + h;
              // (dP - delta) in fp32, rounded once to bf16x2, times P (already bf16x2):
              // FADD2 + F2FP + HMUL2 per pair, no unpacking of P
              const uint64_t dd = f2_add(f2_pack(__uint_as_float(dr[2 * c]),
                                                 __uint_as_float(dr[2 * c + 1])),
                                         h ? f2_pack(-dl.z, -dl.w) : f2_pack(-dl.x, -dl.y));
              float a, b;
              f2_unpack(dd, a, b);
              dk[c] = bf16x2_mul(pkeep[cc * 16 + c], pack_bf16(a, b));
            }
          }
          tmem_st16(dp_addr + half * 96 + cc * 16, dk);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int unit = cc * 4 + u;  // 16-byte unit within this half's 128 B row
            if (AUTOSP_BWD_ABL != 2 && AUTOSP_BWD_ABL != 4)
              sts128(ds_row + ((unit ^ (row & 7)) << 4),
                     make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]));
          }
        }
      };
      if (masked) part2(std::true_type{});
      else part2(std::false_type{});
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive_warp(ds_ready);
      if (threadIdx.x == kSoftWarp0 * 32) BWD_TRACE(8, t);
    }
    // ---- epilogue: dV (WG1) / dK scaled (WG2) straight from TMEM
    if (T > 0) {
      mbar_wait(acc_full, 0);
      tc_fence_after();
      const uint32_t src = tmem + lane_base + (half ? C::DK_COL : C::DV_COL);
      const float sc = half ? p.scale : 1.f;
      if constexpr (SPLIT) {  // GQA split: fp32 partials, finished by bwd_post
        float* acc_row = p.dkv_acc + ((((int64_t)(half ? 0 : 1) * p.B + batch) * p.Hkv + kvh) *
                                      p.S + key) * D;
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t a[32];
          tmem_ld32(src + c, a);
          tmem_wait_ld();
          if (key < p.S) {
#pragma unroll
            for (int t4 = 0; t4 < 8; ++t4)
              red_add_v4(acc_row + c + 4 * t4, a[4 * t4], a[4 * t4 + 1], a[4 * t4 + 2],
                         a[4 * t4 + 3]);
          }
        }
      } else {
      __nv_bfloat16* dst;
      if constexpr (PUSH) {  // fused K2: the row goes to the owner of token `key`
        const int j = min(key, p.S - 1) / p.s_loc;
        const int gh = p.Hq * p.P + (half ? 0 : p.Hkv * p.P) + p.rank * p.Hkv + kvh;
        dst = reinterpret_cast<__nv_bfloat16*>(p.peer_base[j] + p.dst_off) +
              (int64_t)batch * p.d_sb + (int64_t)(key - j * p.s_loc) * p.d_ss +
              (int64_t)gh * p.d_sh;
      } else {
        dst = half ? p.dk + (int64_t)batch * p.dk_sb + (int64_t)kvh * p.dk_sh + (int64_t)key * p.dk_ss
                   : p.dv + (int64_t)batch * p.dv_sb + (int64_t)kvh * p.dv_sh + (int64_t)key * p.dv_ss;
      }
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t a[32];
        tmem_ld32(src + c, a);
        tmem_wait_ld();
        if (key < p.S) {
#pragma unroll
          for (int t4 = 0; t4 < 4; ++t4) {
            uint4 va;
            va.x = pack_bf16(__uint_as_float(a[8 * t4 + 0]) * sc, __uint_as_float(a[8 * t4 + 1]) * sc);
            va.y = pack_bf16(__uint_as_float(a[8 * t4 + 2]) * sc, __uint_as_float(a[8 * t4 + 3]) * sc);
            va.z = pack_bf16(__uint_as_float(a[8 * t4 + 4]) * sc, __uint_as_float(a[8 * t4 + 5]) * sc);
            va.w = pack_bf16(__uint_as_float(a[8 * t4 + 6]) * sc, __uint_as_float(a[8 * t4 + 7]) * sc);
            reinterpret_cast<uint4*>(dst + c)[t4] = va;
          }
        }
      }
      }
    }
  } else if (warp >= kDrainWarp0 && warp < kDrainWarp0 + 4) {
    // ------------------------------------------------------------ dQ drain warpgroup
    // thread = query row.  dQ(t) leaves TMEM 64 columns at a time (one TMEM round trip);
    // the columns are released as soon as the last chunk is in registers (S(t+2) reuses
    // them), then each 32-column chunk is staged through a 128B-swizzled smem slot and
    // TMA-reduce-added (fp32) into the accumulator.  (Per-thread red.global.add.v4 was
    // tried: 2048 L2 atomics per step flood the LSU and stall the softmax's smem stores.)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // query row within the step
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const bool leader = (warp == kDrainWarp0 && lane == 0);
    constexpr int NC = D / 32;  // 32-column chunks
    for (int t = 0; t < T; ++t) {
      const int head = kvh * group + (SPLIT ? (int)(BWD_HEAD_IDX % HS) * gsz : 0) + t / per_head;
      const int q0 = (m_first + t % per_head) * BQ;
      const uint32_t dq_addr = tmem + lane_base + dq_col(t);
      // the slot of chunk 0 was last used two chunks ago: wait for that reduce to have
      // read it BEFORE dQ(t) arrives, off the critical path (dP(t+1) waits for the drain)
      if (leader) bulk_wait_read_n<C::DQS - 1>();
      mbar_wait(dq_full, t & 1);
      if (threadIdx.x == kDrainWarp0 * 32) BWD_TRACE(9, t);
      tc_fence_after();
      // stage one 32-column chunk through a smem slot and TMA-reduce it into dQacc
      auto stage = [&](const uint32_t (&v)[32], int c) {
        const int chunk_id = t * NC + c;
        float* slot = reinterpret_cast<float*>(smem + C::DQ_OFF) + (chunk_id % C::DQS) * (128 * 32);
        if (AUTOSP_BWD_ABL == 1 || AUTOSP_BWD_ABL == 4) return;
        if (leader && c > 0) bulk_wait_read_n<C::DQS - 1>();  // the slot's last reduce has read it
        named_bar_sync(2, 128);
        uint8_t* srow = reinterpret_cast<uint8_t*>(slot) + row * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          sts128(srow + ((u ^ (row & 7)) << 4),
                 make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]));
        fence_proxy_async_smem();
        named_bar_sync(2, 128);
        if (leader) {
          tma_reduce_add_3d(&p.tm_dqacc, slot, c * 32, q0, batch * p.Hq + head);
          bulk_commit();
        }
      };
      if constexpr (NC == 4) {
        // d = 128: dQ(t) sits in the dP columns and dP(t+1) waits for them, so the drain
        // releases them after ONE staging: three chunks in registers, then the fourth
        // into the registers the first one freed
        uint32_t va[32], vb[32], vc[32];
        tmem_ld32(dq_addr + 0, va);
        tmem_ld32(dq_addr + 32, vb);
        tmem_ld32(dq_addr + 64, vc);
        tmem_wait_ld();
        stage(va, 0);
        tmem_ld32(dq_addr + 96, va);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive_warp(dq_empty);
        stage(vb, 1);
        stage(vc, 2);
        stage(va, 3);
      } else
#pragma unroll
      for (int c2 = 0; c2 < NC; c2 += 2) {
        uint32_t v[2][32];
        tmem_ld32(dq_addr + c2 * 32, v[0]);
        if (c2 + 1 < NC) tmem_ld32(dq_addr + (c2 + 1) * 32, v[1]);
        tmem_wait_ld();
        if (c2 + 2 >= NC) {  // all of dQ(t) is in registers: release the TMEM columns
          tc_fence_before();
          mbar_arrive_warp(dq_empty);
        }
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          // (the two staging slots alternate across ALL chunks, also across steps when NC
          // is odd, so wait_group.read 1 always covers the slot's previous reduce)
          if (c2 + cc < NC) stage(v[cc], c2 + cc);
        }
      }
      if (threadIdx.x == kDrainWarp0 * 32) BWD_TRACE(10, t);
    }
    if (leader) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kAllocWarp) tmem_dealloc<512>(tmem);
  // pushed dK/dV rows: visible system-wide before bwd_post publishes the arrival (the
  // CTA barrier above orders every thread's stores before this cumulative fence)
  if (PUSH && threadIdx.x == 0) __threadfence_system();
}


// ---------------------------------------------------------------------------- pre / post
struct PrePost {
  const __nv_bfloat16* o;
  const __nv_bfloat16* d_o;
  __nv_bfloat16* dq;
  int64_t o_sb, o_sh, o_ss, do_sb, do_sh, do_ss, dq_sb, dq_sh, dq_ss;
  float* dqacc;
  float* delta;
  const float* lse;  // forward LSE (natural log)
  float* nlse2;      // -lse * log2(e): the exp2 argument offset the softmax-grad warps use
  int delta_given;   // 1: delta supplied by the caller (no O needed), only dQacc / nlse2
  int Hq, S, D;
  int64_t rows;
  float scale;
  // push: dq rows go to the token owner's packed gradient (global head rank*Hq + h) and
  // the last CTA publishes the call's arrival (flags.cuh)
  int push, P, rank, s_loc;
  int64_t dst_off, d_sb, d_ss, d_sh;
  char* peer_base[AUTOSP_MAX_WORLD];
  uint32_t* peer_flags[AUTOSP_MAX_WORLD];
  uint32_t epoch, check;
  // GQA split: dK / dV finished here from the fp32 partials (rows after the dQ rows)
  int Hkv;
  int64_t rows_kv;  // B * Hkv * S (0 without the split)
  const float* dkv_acc;
  __nv_bfloat16 *dk, *dv;
  int64_t dk_sb, dk_sh, dk_ss, dv_sb, dv_sh, dv_ss;
};

// delta[row] = sum_d dO*O ; nlse2[row] = -lse[row] * log2(e) ; dqacc[row, :] = 0.
// lanes_per_row = D/8 (one 16B vector each).
__global__ void bwd_pre_kernel(const __grid_constant__ PrePost a) {
  const int lpr = a.D / 8;
  const int rpw = 32 / lpr;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t row = warp * rpw + lane / lpr;
  const int sub = lane % lpr;
  float acc = 0.f;
  if (row < a.rows && !a.delta_given) {
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
  }
  if (row < a.rows) {
    float4* z = reinterpret_cast<float4*>(a.dqacc + row * a.D + sub * 8);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int off = lpr / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (row < a.rows && sub == 0) {
    if (!a.delta_given) a.delta[row] = acc;
    a.nlse2[row] = -a.lse[row] * 1.4426950408889634f;
  }
}

__global__ void bwd_post_kernel(const __grid_constant__ PrePost a) {
  const int lpr = a.D / 8;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid / lpr;
  const int sub = (int)(gid % lpr);
  if (row >= a.rows && row < a.rows + 2 * a.rows_kv) {  // GQA-split dK / dV rows
    const int64_t r2 = row - a.rows;
    const int which = (int)(r2 / a.rows_kv);               // 0 dK (scaled), 1 dV
    const int64_t rr = r2 - which * a.rows_kv;
    const int key = (int)(rr % a.S);
    const int64_t bh = rr / a.S;
    const int kvh = (int)(bh % a.Hkv);
    const int64_t bi = bh / a.Hkv;
    const float sc = which == 0 ? a.scale : 1.f;
    const float4* src = reinterpret_cast<const float4*>(a.dkv_acc + r2 * a.D + sub * 8);
    const float4 x = src[0], y = src[1];
    uint4 v;
    v.x = pack_bf16(x.x * sc, x.y * sc);
    v.y = pack_bf16(x.z * sc, x.w * sc);
    v.z = pack_bf16(y.x * sc, y.y * sc);
    v.w = pack_bf16(y.z * sc, y.w * sc);
    __nv_bfloat16* dst;
    if (a.push) {
      const int j = key / a.s_loc;
      const int gh = a.Hq * a.P + (which ? a.Hkv * a.P : 0) + a.rank * a.Hkv + kvh;
      dst = reinterpret_cast<__nv_bfloat16*>(a.peer_base[j] + a.dst_off) + bi * a.d_sb +
            (int64_t)(key - j * a.s_loc) * a.d_ss + (int64_t)gh * a.d_sh;
    } else {
      dst = which == 0 ? a.dk + bi * a.dk_sb + kvh * a.dk_sh + (int64_t)key * a.dk_ss
                       : a.dv + bi * a.dv_sb + kvh * a.dv_sh + (int64_t)key * a.dv_ss;
    }
    *reinterpret_cast<uint4*>(dst + sub * 8) = v;
  }
  if (row < a.rows) {
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
    if (a.push) {  // lanes of one row store its D*2 contiguous bytes together
      const int j = q / a.s_loc;
      *reinterpret_cast<uint4*>(
          reinterpret_cast<__nv_bfloat16*>(a.peer_base[j] + a.dst_off) + bi * a.d_sb +
          (int64_t)(q - j * a.s_loc) * a.d_ss + (int64_t)(a.rank * a.Hq + h) * a.d_sh + sub * 8) = v;
    } else {
      *reinterpret_cast<uint4*>(a.dq + bi * a.dq_sb + h * a.dq_sh + (int64_t)q * a.dq_ss +
                                sub * 8) = v;
    }
  }
  if (a.push) publish_arrival(a.peer_flags, a.P, a.rank, a.epoch, a.check, gridDim.x);
}

// GQA split of small grids: two CTAs per (key tile, kv head) when the grid would not fill
// two waves of SMs (e.g. SP = 8 with one kv head per rank: 256 CTAs for 148 SMs, the
// heaviest causal CTA then bounds the kernel).  AUTOSP_BWD_HSPLIT=1 disables, =2 forces.
inline int choose_hsplit(int B, int Hq, int Hkv, int S) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("AUTOSP_BWD_HSPLIT");
    mode = e ? atoi(e) : 0;
  }
  const int group = Hq / Hkv;
  if (group % 2 || mode == 1) return 1;
  if (mode == 2) return 2;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t ctas = (int64_t)((S + BK - 1) / BK) * Hkv * B;
  return ctas < 2LL * sms ? 2 : 1;
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
           int causal, const float* delta_in, const autosp_push_spec* push,
           cudaStream_t stream) {
  using C = Cfg<D>;
  float* dqacc = static_cast<float*>(ws);
  float* delta = delta_in ? const_cast<float*>(delta_in) : dqacc + (size_t)B * Hq * S * D;
  float* nlse2 = dqacc + (size_t)B * Hq * S * D + (size_t)B * Hq * S;
  const int hsplit = choose_hsplit(B, Hq, Hkv, S);
  float* dkv_acc = hsplit > 1 ? nlse2 + (size_t)B * Hq * S : nullptr;
  PrePost a{};
  a.o = static_cast<const __nv_bfloat16*>(o.ptr);
  a.d_o = static_cast<const __nv_bfloat16*>(d_o.ptr);
  a.dq = static_cast<__nv_bfloat16*>(const_cast<void*>(dq.ptr));
  a.o_sb = o.stride_b; a.o_sh = o.stride_h; a.o_ss = o.stride_s;
  a.do_sb = d_o.stride_b; a.do_sh = d_o.stride_h; a.do_ss = d_o.stride_s;
  a.dq_sb = dq.stride_b; a.dq_sh = dq.stride_h; a.dq_ss = dq.stride_s;
  a.dqacc = dqacc;
  a.delta = delta;
  a.lse = lse;
  a.nlse2 = nlse2;
  a.delta_given = delta_in ? 1 : 0;
  a.Hq = Hq;
  a.S = S;
  a.D = D;
  a.rows = (int64_t)B * Hq * S;
  a.scale = scale;
  a.Hkv = Hkv;
  a.rows_kv = hsplit > 1 ? (int64_t)B * Hkv * S : 0;
  a.dkv_acc = dkv_acc;
  a.dk = static_cast<__nv_bfloat16*>(const_cast<void*>(dk.ptr));
  a.dv = static_cast<__nv_bfloat16*>(const_cast<void*>(dv.ptr));
  a.dk_sb = dk.stride_b; a.dk_sh = dk.stride_h; a.dk_ss = dk.stride_s;
  a.dv_sb = dv.stride_b; a.dv_sh = dv.stride_h; a.dv_ss = dv.stride_s;
  if (hsplit > 1)
    cudaMemsetAsync(dkv_acc, 0, (size_t)2 * B * Hkv * S * D * sizeof(float), stream);
  if (push) {
    a.push = 1;
    a.P = push->world;
    a.rank = push->rank;
    a.s_loc = S / push->world;
    a.dst_off = push->dst_offset;
    a.d_sb = push->dst_stride_b;
    a.d_ss = push->dst_stride_s;
    a.d_sh = push->dst_stride_h;
    for (int j = 0; j < push->world; ++j) {
      a.peer_base[j] = static_cast<char*>(push->peer_base[j]);
      a.peer_flags[j] = push->peer_flags[j];
    }
    a.epoch = push->epoch;
    a.check = autosp_push_check(push, Hq + 2 * Hkv);
  }
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
  p.lse_tma = (S % 4 == 0) && make_map_rows_f32(&p.tm_lse, nlse2, B * Hq, S) &&
              make_map_rows_f32(&p.tm_dlt, delta, B * Hq, S);
  if (!ok) {
    autosp_set_error("attn_bwd: cuTensorMapEncodeTiled failed (alignment/strides?)");
    return AUTOSP_ERR_VALIDATION;
  }
  p.lse = nlse2;  // the softmax-grad warps read -lse*log2(e)
  p.delta = delta;
  p.dqacc = dqacc;
  p.trace = g_bwd_trace;
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
  p.hsplit = hsplit;
  p.dkv_acc = dkv_acc;
  if (push) {
    p.push = 1;
    p.P = a.P;
    p.rank = a.rank;
    p.s_loc = a.s_loc;
    p.dst_off = a.dst_off;
    p.d_sb = a.d_sb;
    p.d_ss = a.d_ss;
    p.d_sh = a.d_sh;
    for (int j = 0; j < a.P; ++j) p.peer_base[j] = a.peer_base[j];
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_bwd_kernel<D, false, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(attn_bwd_kernel<D, true, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(attn_bwd_kernel<D, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(attn_bwd_kernel<D, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr_set = true;
  }
  const dim3 grid = causal_grid(AUTOSP_BWD_LPT, p.n_ktiles, Hkv * hsplit, B);
  if (push && hsplit > 1) attn_bwd_kernel<D, true, true><<<grid, kThreads, C::SMEM, stream>>>(p);
  else if (push) attn_bwd_kernel<D, true, false><<<grid, kThreads, C::SMEM, stream>>>(p);
  else if (hsplit > 1) attn_bwd_kernel<D, false, true><<<grid, kThreads, C::SMEM, stream>>>(p);
  else attn_bwd_kernel<D, false, false><<<grid, kThreads, C::SMEM, stream>>>(p);
  {
    const int64_t threads = (a.rows + 2 * a.rows_kv) * (D / 8);
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

extern "C" size_t autosp_attn_bwd_workspace_bytes(int b, int hq, int hkv, int s, int d) {
  if (b < 1 || hq < 1 || hkv < 1 || s < 1 || d < 1 || hq % hkv) return 0;
  size_t f = (size_t)b * hq * s * (d + 2);  // dQ acc + delta + -lse*log2(e)
  if (autosp::bwd::choose_hsplit(b, hq, hkv, s) > 1)
    f += (size_t)2 * b * hkv * s * d;  // GQA-split dK / dV partials
  return f * sizeof(float);
}

static int attn_bwd_impl(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                         autosp_attn_tensor o, const float* delta, autosp_attn_tensor d_o,
                         const float* lse, autosp_attn_tensor dq, autosp_attn_tensor dk,
                         autosp_attn_tensor dv, void* workspace, int b, int hq, int hkv, int s,
                         int d, float scale, int causal, const autosp_push_spec* push,
                         void* stream);
int autosp_internal_handshake(uint32_t* const* flags, int world, int rank, uint32_t epoch,
                              cudaStream_t stream);

extern "C" int autosp_attn_bwd(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                               autosp_attn_tensor o, autosp_attn_tensor d_o, const float* lse,
                               autosp_attn_tensor dq, autosp_attn_tensor dk,
                               autosp_attn_tensor dv, void* workspace, int b, int hq, int hkv,
                               int s, int d, float scale, int causal, void* stream) {
  int rc;
  if ((rc = autosp_check_attn_tensor(o, "o"))) return rc;
  return attn_bwd_impl(q, k, v, o, nullptr, d_o, lse, dq, dk, dv, workspace, b, hq, hkv, s, d,
                       scale, causal, nullptr, stream);
}

extern "C" int autosp_attn_bwd_delta(autosp_attn_tensor q, autosp_attn_tensor k,
                                     autosp_attn_tensor v, const float* delta,
                                     autosp_attn_tensor d_o, const float* lse,
                                     autosp_attn_tensor dq, autosp_attn_tensor dk,
                                     autosp_attn_tensor dv, void* workspace, int b, int hq,
                                     int hkv, int s, int d, float scale, int causal,
                                     void* stream) {
  if (!delta || (reinterpret_cast<uintptr_t>(delta) & 15)) {
    autosp_set_error("attn_bwd_delta: delta must be non-null and 16-byte aligned");
    return AUTOSP_ERR_VALIDATION;
  }
  return attn_bwd_impl(q, k, v, q /* unused */, delta, d_o, lse, dq, dk, dv, workspace, b, hq,
                       hkv, s, d, scale, causal, nullptr, stream);
}

extern "C" int autosp_attn_bwd_push(autosp_attn_tensor q, autosp_attn_tensor k,
                                    autosp_attn_tensor v, const float* delta,
                                    autosp_attn_tensor d_o, const float* lse, void* workspace,
                                    int b, int hq, int hkv, int s, int d, float scale,
                                    int causal, const autosp_push_spec* push, void* stream) {
  if (!delta || (reinterpret_cast<uintptr_t>(delta) & 15)) {
    autosp_set_error("attn_bwd_push: delta must be non-null and 16-byte aligned");
    return AUTOSP_ERR_VALIDATION;
  }
  if (!push || push->world < 1 || push->world > AUTOSP_MAX_WORLD || push->rank < 0 ||
      push->rank >= push->world || !push->peer_base || !push->peer_flags) {
    autosp_set_error("attn_bwd_push: bad push spec");
    return AUTOSP_ERR_VALIDATION;
  }
  if (s % push->world) {
    autosp_set_error("attn_bwd_push: sequence %d not divisible by world size %d", s,
                     push->world);
    return AUTOSP_ERR_VALIDATION;
  }
  if (push->dst_offset % 16 || push->dst_stride_b % 8 || push->dst_stride_s % 8 ||
      push->dst_stride_h % 8 || push->dst_stride_h < d) {
    autosp_set_error("attn_bwd_push: destination offset/strides must be 16-byte multiples");
    return AUTOSP_ERR_VALIDATION;
  }
  for (int j = 0; j < push->world; ++j)
    if (!push->peer_base[j] || !push->peer_flags[j] ||
        (reinterpret_cast<uintptr_t>(push->peer_base[j]) & 15)) {
      autosp_set_error("attn_bwd_push: peer %d base/flags null or misaligned", j);
      return AUTOSP_ERR_VALIDATION;
    }
  autosp_attn_tensor none{};
  none.ptr = q.ptr;  // dq/dk/dv are never written locally (validated shape-only)
  none.stride_b = q.stride_b; none.stride_h = q.stride_h; none.stride_s = q.stride_s;
  if (push->world > 1) {
    int rc = autosp_internal_handshake(push->peer_flags, push->world, push->rank, push->epoch,
                                       static_cast<cudaStream_t>(stream));
    if (rc) {
      autosp_set_error("attn_bwd_push: handshake launch failed");
      return rc;
    }
  }
  return attn_bwd_impl(q, k, v, q /* unused */, delta, d_o, lse, none, none, none, workspace, b,
                       hq, hkv, s, d, scale, causal, push, stream);
}

static int attn_bwd_impl(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                         autosp_attn_tensor o, const float* delta, autosp_attn_tensor d_o,
                         const float* lse, autosp_attn_tensor dq, autosp_attn_tensor dk,
                         autosp_attn_tensor dv, void* workspace, int b, int hq, int hkv, int s,
                         int d, float scale, int causal, const autosp_push_spec* push,
                         void* stream) {
  if (b < 1 || hq < 1 || hkv < 1 || s < 1 || hq % hkv) {
    autosp_set_error("attn_bwd: bad shape b=%d hq=%d hkv=%d s=%d", b, hq, hkv, s);
    return AUTOSP_ERR_VALIDATION;
  }
  int rc;
  if ((rc = autosp_check_attn_tensor(q, "q")) || (rc = autosp_check_attn_tensor(k, "k")) ||
      (rc = autosp_check_attn_tensor(v, "v")) ||
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
                                     scale, causal, delta, push, st);
    case 64:
      return autosp::bwd::launch<64>(q, k, v, o, d_o, lse, dq, dk, dv, workspace, b, hq, hkv, s,
                                     scale, causal, delta, push, st);
    case 128:
      return autosp::bwd::launch<128>(q, k, v, o, d_o, lse, dq, dk, dv, workspace, b, hq, hkv, s,
                                      scale, causal, delta, push, st);
    default:
      autosp_set_error("attn_bwd: head_dim %d unsupported (32, 64, 128)", d);
      return AUTOSP_ERR_UNSUPPORTED;
  }
}

// Debug-only (tools/bwd_trace.py): record a per-step timeline of CTA (0,0,0).
extern "C" AUTOSP_API int autosp_debug_set_bwd_trace(long long* dev_buf) {
  autosp::bwd::g_bwd_trace = dev_buf;
  return AUTOSP_OK;
}

int autosp_preload_bwd() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<32, false, false>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<32, true, false>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<32, false, true>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<32, true, true>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<64, false, false>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<64, true, false>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<64, false, true>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<64, true, true>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<128, false, false>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<128, true, false>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<128, false, true>);
  cudaFuncGetAttributes(&a, autosp::bwd::attn_bwd_kernel<128, true, true>);
  cudaFuncGetAttributes(&a, autosp::bwd::bwd_pre_kernel);
  cudaFuncGetAttributes(&a, autosp::bwd::bwd_post_kernel);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
