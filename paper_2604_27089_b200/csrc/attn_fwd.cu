// K3: causal flash-attention forward on the local head block over the FULL gathered
// sequence (the AttentionCore after the seq->head all-to-all; reference semantics
// executor.py:132-142 / lowering.py:82-122: softmax(q k^T / sqrt(d) + M) v with M the
// strictly-upper-triangular mask), written for sm_100a:
//
//  * one CTA = one (batch, q head, 256-query block) processed as two 128-row Q tiles that
//    ping-pong on the tensor core (while softmax works on tile 0, the MMA runs tile 1);
//  * warp 0: TMA producer (Q once, then a K/V ring of kStages 128-key tiles, 128B swizzle);
//  * warp 1: single-thread tcgen05.mma issuer: S_i = Q_i K^T (SS, M=128,N=128) into TMEM,
//    O_i += P_i V (TS: P read straight from TMEM, V MN-major from smem);
//  * warps 4-7 / 8-11: softmax warpgroups, one query row per thread (TMEM lane), online
//    softmax in the log2 domain with lazy O rescaling (only when the row max grows by
//    more than 2^8), P written back to TMEM as bf16 aliasing S;
//  * causal: KV tiles above the diagonal are never loaded; only the diagonal tile masks;
//  * outputs O (bf16) and the natural-log LSE per row (what sp_ac saves instead of the
//    O(s^2) probabilities, SURVEY §0 finding 3).
#include <cmath>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "../../include/autosp.h"
#include "flags.cuh"
#include "ptx.cuh"
#include "tma.cuh"

extern "C" void autosp_set_error(const char* fmt, ...);

#ifndef AUTOSP_FWD_EMU
#define AUTOSP_FWD_EMU 1  // exps per 8 on the FMA pipe for d <= 64 (A/B: 1 > 0 > 2 > 3)
#endif
#ifndef AUTOSP_FWD_LATE_ODONE
#define AUTOSP_FWD_LATE_ODONE 1  // optimistic pass: wait for PV(j-1) only before the first P store (A/B: +2.3 %)
#endif
#ifndef AUTOSP_FWD_RESCALE_T
#define AUTOSP_FWD_RESCALE_T 8  // lazy rescale / optimistic-pass threshold (log2 units)
#endif
#ifndef AUTOSP_FWD_KVRING64
#define AUTOSP_FWD_KVRING64 98304  // K/V ring bytes for d <= 64 (3 stages of 128 keys at d = 64)
#endif
#ifndef AUTOSP_FWD_MMA2
#define AUTOSP_FWD_MMA2 1  // one MMA-issuing warp per Q tile for d <= 64 (A/B: +1.5 % at
#endif                     // d = 64; -11 % at d = 128, where it stays off)
#ifndef AUTOSP_FWD_EARLY_K
#define AUTOSP_FWD_EARLY_K 1  // wait for K_{j+1} before s_free (off the hand-off path)
#endif
#ifndef AUTOSP_FWD_LATE_V
#define AUTOSP_FWD_LATE_V 1  // d = 128: MMA warp checks V_j just before PV(j), not at the top
                             // of step j (A/B: +1.3 % at d = 128, -0.7 % at d = 64: d > 64 only)
#endif
#ifndef AUTOSP_FWD_MMA4
#define AUTOSP_FWD_MMA4 1  // d <= 64: one MMA stream per SMSP (see Cfg); A/B: +3.4 % at d = 64
#endif
#ifndef AUTOSP_FWD_MMA4_KROLE
#define AUTOSP_FWD_MMA4_KROLE 0  // MMA4: the QK stream (0 or 2) that issues the K loads
#endif
#ifndef AUTOSP_FWD_MMA4_VROLE
#define AUTOSP_FWD_MMA4_VROLE 2  // MMA4: the QK stream (0 or 2) that issues the V loads (A/B: 2 > 0)
#endif
#ifndef AUTOSP_FWD_KVRING64_MMA4
#define AUTOSP_FWD_KVRING64_MMA4 163840  // MMA4: 5 K/V stages (loads issued one tile later)
#endif
#ifndef AUTOSP_FWD_LPT
#define AUTOSP_FWD_LPT 1  // LPT grid layout (ptx.cuh; A/B: +1.6 % full shape, +37 % at 4 heads x 16K)
#endif
#ifndef AUTOSP_FWD_EMU128
#define AUTOSP_FWD_EMU128 2  // exps per 8 on the FMA pipe for d = 128
#endif

namespace autosp {
namespace fwd {

constexpr int BM = 128;  // query rows per tile
constexpr int kSoftmaxWarp0 = 0;   // warps 4i..4i+3: softmax of Q tile i
// Tile shape (build-time, swept with tools/attn_bench.py): 64-key tiles (3 x 64 for
// d <= 64, or 2 x 64 with separate P buffers for d = 128) measured 25 % slower than
// 2 Q tiles x 128 keys -- the per-tile hand-off chain (S -> softmax -> P -> PV) is paid
// twice as often -- so 2 x 128 is the default.
#ifndef AUTOSP_FWD_NQ64
#define AUTOSP_FWD_NQ64 2     // Q tiles per CTA for d <= 64
#endif
#ifndef AUTOSP_FWD_BN64
#define AUTOSP_FWD_BN64 128   // keys per KV tile for d <= 64
#endif
#ifndef AUTOSP_FWD_BN128
#define AUTOSP_FWD_BN128 128  // keys per KV tile for d = 128
#endif

template <int D>
struct Cfg {
  // NQ Q tiles of 128 rows per CTA ping-pong on the tensor core, one softmax warpgroup
  // each; KV tiles of BN keys (see the tile-shape note above).
  static constexpr int NQ = D == 128 ? 2 : AUTOSP_FWD_NQ64;
  static constexpr int BN = D == 128 ? AUTOSP_FWD_BN128 : AUTOSP_FWD_BN64;
  static constexpr int NH = BN / 64;                        // 64-column score chunks
  static constexpr int kThreads = 32 * (4 * NQ + 4);
  // Warp roles.  The issue arbiter favours HIGHER warp ids, so the latency-critical
  // single-thread producers (TMA, MMA) get the top ids and are never starved by the
  // instruction-heavy softmax warpgroups (whole, aligned warpgroups for TMEM lanes).
  static constexpr int kAllocWarp = 4 * NQ;
  static constexpr int kTmaWarp = 4 * NQ + ((AUTOSP_FWD_MMA4 && NQ == 2 && D <= 64) ? 0 : 2);
  static constexpr int kMmaWarp = 4 * NQ + 3;
  // AUTOSP_FWD_MMA2 (NQ = 2): warp 4NQ+1 issues tile 0's MMAs, kMmaWarp tile 1's -- each
  // tile's QK / PV wait only on its own softmax; the K/V stages are released by both
  static constexpr bool MMA2 = AUTOSP_FWD_MMA2 && !AUTOSP_FWD_MMA4 && NQ == 2 && D <= 64;
  static constexpr int kMmaWarp2 = 4 * NQ + 1;
  // AUTOSP_FWD_MMA4 (NQ = 2, d <= 64): the four MMA streams QK_0, PV_0, QK_1, PV_1 issued by
  // warps 4NQ+0..3 -- one per SMSP, so the issue stalls of tcgen05.mma (it blocks while the
  // pipe is busy) fall evenly on the softmax warps; warp 4NQ also allocates TMEM and runs
  // the TMA loads (each load issued once the stage's previous tile is released)
  static constexpr bool MMA4 = AUTOSP_FWD_MMA4 && NQ == 2 && D <= 64;
  static constexpr int SW = (D * 2 >= 128) ? 128 : D * 2;  // swizzle bytes
  static constexpr int CE = SW / 2;                         // elements per swizzle chunk
  static constexpr int NCH = D / CE;                        // chunks per row
  static constexpr int TILE_BYTES = BM * D * 2;             // Q tile: 128 x D bf16
  static constexpr int KTILE = BN * D * 2;                  // K / V tile: BN x D bf16
  static constexpr int KV_RING = D == 128 ? 131072
                                : ((AUTOSP_FWD_MMA4 && NQ == 2) ? AUTOSP_FWD_KVRING64_MMA4
                                                                : AUTOSP_FWD_KVRING64);
  static constexpr int kStagesRaw = KV_RING / (2 * KTILE);
  static constexpr int kStages = kStagesRaw < 2 ? 2 : (kStagesRaw > 8 ? 8 : kStagesRaw);
  // exps per 8 computed by the FMA-pipe polynomial instead of MUFU (MUFU is the
  // bottleneck when the tile's MMA work is small: d = 32 / 64)
  static constexpr int kEmuPer8 = D == 128 ? AUTOSP_FWD_EMU128 : AUTOSP_FWD_EMU;
  static constexpr int LAYOUT = SW == 128 ? 2 : (SW == 64 ? 4 : 6);
  static constexpr int SBO = 8 * SW;  // 8-row swizzle atom
  // smem: Q[NQ] | K[kStages] | V[kStages] | barriers
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = NQ * TILE_BYTES;
  static constexpr int V_OFF = K_OFF + kStages * KTILE;
  static constexpr int BAR_OFF = V_OFF + kStages * KTILE;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;  // + alignment slack
  static_assert(SMEM <= 232448, "shared memory budget");
  static constexpr uint32_t TMEM_COLS = 512;
  // TMEM: S_0..S_{NQ-1} (BN fp32 cols each) | P_i (bf16, BN/2 cols) | O_i (D cols).
  // Separate P buffers (SEP_P) let S_i(j+1) = Q_i K^T be issued as soon as the softmax
  // has READ S_i(j), overlapping the rest of the softmax and PV_i(j); without room for
  // them P aliases S (only the old 128-key d = 128 layout).
  static constexpr bool SEP_P = NQ * (BN + BN / 2 + D) <= (int)TMEM_COLS;
  static constexpr uint32_t S_COL = 0;                         // S_i at i*BN
  static constexpr uint32_t P_COL = SEP_P ? NQ * BN : 0;       // P_i at P_COL + i*P_STRIDE
  static constexpr uint32_t P_STRIDE = SEP_P ? BN / 2 : BN;
  static constexpr uint32_t O_COL = SEP_P ? NQ * (BN + BN / 2) : NQ * BN;  // O_i at O_COL + i*D
  static_assert(O_COL + NQ * D <= TMEM_COLS, "TMEM budget");
  static_assert(BN == 64 || BN == 128, "KV tile");
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v;
  __nv_bfloat16* o;
  int64_t o_sb, o_sh, o_ss;
  float* lse;
  int B, Hq, Hkv, S;
  float scale_log2;
  int causal;
  int n_qblk;
  long long* trace;  // debug timeline of the heaviest CTA (nullptr in production)
  // fused head->seq all-to-all of O (autosp_attn_fwd_push); push == 0: local O only
  int push, P, rank, s_loc;
  int64_t dst_off, d_sb, d_ss, d_sh;  // bytes / elements
  char* peer_base[AUTOSP_MAX_WORLD];
  uint32_t* peer_flags[AUTOSP_MAX_WORLD];
  uint32_t epoch, check;
};
constexpr int kTraceSteps = 64;
#define FWD_TRACE_RAW(ev, t)                                                               \
  do {                                                                                     \
    if (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (t) < kTraceSteps) \
      p.trace[(ev) * kTraceSteps + (t)] = clock64();                                       \
  } while (0)
#ifndef AUTOSP_FWD_TRACE_SKEW
#define AUTOSP_FWD_TRACE_SKEW 0  // tools only (fwd_skew_trace.py): per-warp S release / P arrival
#endif
#if AUTOSP_FWD_TRACE_SKEW
#define FWD_TRACE(ev, t) do { if ((ev) == 4 || (ev) == 5) FWD_TRACE_RAW(ev, t); } while (0)
#define FWD_TRACE_SKEW(base, t) do { if (lane == 0 && warp < 4) FWD_TRACE_RAW((base) + warp, t); } while (0)
#else
#define FWD_TRACE(ev, t) FWD_TRACE_RAW(ev, t)
#define FWD_TRACE_SKEW(base, t) do { } while (0)
#endif
long long* g_fwd_trace = nullptr;

// byte offset >> 4 of K-step kk inside a K-major tile of ROWS rows stored as NCH swizzled
// chunks of [ROWS x SW bytes] (added to the descriptor's start address)
template <int D, int ROWS>
__host__ __device__ constexpr uint64_t kmajor_off(int kk) {
  return (uint64_t)((((kk * 16) / Cfg<D>::CE) * (ROWS * Cfg<D>::SW) + ((kk * 16) % Cfg<D>::CE) * 2) >> 4);
}

template <int D>
__global__ void __launch_bounds__(Cfg<D>::kThreads, 1) attn_fwd_kernel(const __grid_constant__ Params p) {
  using C = Cfg<D>;
  constexpr int NQ = C::NQ, BN = C::BN;
  constexpr int kAllocWarp = C::kAllocWarp, kTmaWarp = C::kTmaWarp, kMmaWarp = C::kMmaWarp;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + C::kStages;
  uint64_t* v_full = k_empty + C::kStages;
  uint64_t* v_empty = v_full + C::kStages;
  uint64_t* s_full = v_empty + C::kStages;  // [NQ]
  uint64_t* p_full = s_full + NQ;           // [NQ]
  uint64_t* o_done = p_full + NQ;           // [NQ]
  uint64_t* s_free = o_done + NQ;           // [NQ] softmax finished reading S_i (SEP_P)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_free + NQ);

  const int warp = warp_id();
  const int lane = lane_id();
  const int qblk = p.n_qblk - 1 - (int)AUTOSP_BLOCK_RANK(AUTOSP_FWD_LPT);  // heaviest causal blocks first
  const int head = AUTOSP_BLOCK_HEAD(AUTOSP_FWD_LPT);
  const int batch = blockIdx.z;
  const int kvhead = head / (p.Hq / p.Hkv);
  const int q0 = qblk * NQ * BM;
  const int n_kv_total = (p.S + BN - 1) / BN;
  int n_tiles[NQ];
  int n_max = 0;
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    const int last_row = min(q0 + (i + 1) * BM, p.S) - 1;
    n_tiles[i] = p.causal ? min(last_row / BN + 1, n_kv_total) : n_kv_total;
    if (q0 + i * BM >= p.S) n_tiles[i] = 0;
    n_max = max(n_max, n_tiles[i]);
  }

  if (warp == kTmaWarp && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, (C::MMA2 || C::MMA4) ? 2 : 1);
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, (C::MMA2 || C::MMA4) ? 2 : 1);
    }
    for (int i = 0; i < NQ; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 4);   // one arrival per softmax warp
      mbar_init(o_done + i, 1);
      mbar_init(s_free + i, 4);
    }
    fence_mbar_init();
    tma_prefetch_desc(&p.tm_q);
    tma_prefetch_desc(&p.tm_k);
    tma_prefetch_desc(&p.tm_v);
  }
  if (warp == kAllocWarp) tmem_alloc<C::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t sq = smem_u32(smem + C::Q_OFF);
  const uint32_t sk = smem_u32(smem + C::K_OFF);
  const uint32_t sv = smem_u32(smem + C::V_OFF);

  if (C::MMA4 && warp >= 4 * NQ) {
    // ------------------------------------------------------------ MMA4 producers
    const int role = warp - 4 * NQ;  // 0: loads + QK_0, 1: PV_0, 2: QK_1, 3: PV_1
    const int i = role >> 1;
    const bool is_qk = (role & 1) == 0;
    if (n_max > 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(BM, D, 0, 1);
      const uint64_t pol_kv = policy_evict_last();
      auto load_k = [&](int L) {  // lane 0
        const int st = L % C::kStages;
        if (L >= C::kStages) mbar_wait(k_empty + st, ((L / C::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(k_full + st, C::KTILE);
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(smem + C::K_OFF + st * C::KTILE + c * BN * C::SW, &p.tm_k, k_full + st,
                      c * C::CE, L * BN, kvhead, batch, pol_kv);
      };
      auto load_v = [&](int L) {  // lane 0
        const int st = L % C::kStages;
        if (L >= C::kStages) mbar_wait(v_empty + st, ((L / C::kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(v_full + st, C::KTILE);
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(smem + C::V_OFF + st * C::KTILE + c * BN * C::SW, &p.tm_v, v_full + st,
                      c * C::CE, L * BN, kvhead, batch, pol_kv);
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) tc_commit(bar);
        __syncwarp();
      };
      if (role == 0) {
        if (lane == 0) {
          const uint64_t pol_q = policy_evict_first();
          int nq_live = 0;
          for (int t = 0; t < NQ; ++t) nq_live += (q0 + t * BM < p.S) ? 1 : 0;
          mbar_arrive_expect_tx(q_full, nq_live * C::TILE_BYTES);
          for (int t = 0; t < nq_live; ++t)
            for (int c = 0; c < C::NCH; ++c)
              tma_load_4d(smem + C::Q_OFF + t * C::TILE_BYTES + c * BM * C::SW, &p.tm_q, q_full,
                          c * C::CE, q0 + t * BM, head, batch, pol_q);
          for (int L = 0; L < C::kStages && L < n_max; ++L) {
            load_k(L);
            load_v(L);
          }
        }
        __syncwarp();
      }
      if (is_qk) {
        auto issue_qk = [&](int j) {
          const int st = j % C::kStages;
          const uint64_t da = make_smem_desc(sq + i * C::TILE_BYTES, 16, C::SBO, C::LAYOUT);
          const uint64_t db = make_smem_desc(sk + st * C::KTILE, 16, C::SBO, C::LAYOUT);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              mma_ss(tmem + C::S_COL + i * BN, da + kmajor_off<D, BM>(kk),
                     db + kmajor_off<D, BN>(kk), idesc_qk, kk > 0);
            tc_commit(s_full + i);
          }
          __syncwarp();
        };
        mbar_wait(q_full, 0);
        mbar_wait(k_full + 0, 0);
        tc_fence_after();
        if (n_tiles[i] > 0) issue_qk(0);
        commit(k_empty + 0);
        for (int j = 0; j < n_max; ++j) {
          // K of tile j + kStages - 1 into the stage tile j - 1 used (released by both QK
          // streams long ago); V follows after this step's QK
          const int L = j + C::kStages - 1;
          if (role == AUTOSP_FWD_MMA4_KROLE && j >= 1 && L < n_max) {
            if (lane == 0) load_k(L);
            __syncwarp();
          }
          if (j + 1 < n_max) {
            const int st1 = (j + 1) % C::kStages;
            mbar_wait(k_full + st1, ((j + 1) / C::kStages) & 1);
            tc_fence_after();
            if (j + 1 < n_tiles[i]) {
              mbar_wait(s_free + i, j & 1);  // S_i(j) read: S_i(j+1) may overwrite it
              tc_fence_after();
              issue_qk(j + 1);
            }
            commit(k_empty + st1);
          }
          if (role == AUTOSP_FWD_MMA4_VROLE && j >= 1 && L < n_max) {
            if (lane == 0) load_v(L);
            __syncwarp();
          }
        }
      } else {
        for (int j = 0; j < n_max; ++j) {
          const int st = j % C::kStages;
          mbar_wait(v_full + st, (j / C::kStages) & 1);
          if (j < n_tiles[i]) {
            mbar_wait(p_full + i, j & 1);
            tc_fence_after();
            const uint64_t dv = make_smem_desc(sv + st * C::KTILE, BN * C::SW, C::SBO, C::LAYOUT);
            const uint32_t pa = tmem + C::P_COL + i * C::P_STRIDE;
            const uint32_t oa = tmem + C::O_COL + i * D;
            const uint32_t acc0 = j > 0 ? 1u : 0u;
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < BN / 16; ++kk)
                mma_ts(oa, pa + kk * 8, dv + (uint64_t)((kk * 16 * C::SW) >> 4), idesc_pv,
                       kk > 0 ? 1u : acc0);
              tc_commit(o_done + i);
            }
            __syncwarp();
          }
          commit(v_empty + st);
        }
      }
    }
  } else if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && n_max > 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      int nq_live = 0;
      for (int i = 0; i < NQ; ++i) nq_live += (q0 + i * BM < p.S) ? 1 : 0;
      mbar_arrive_expect_tx(q_full, nq_live * C::TILE_BYTES);
      for (int i = 0; i < nq_live; ++i)
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(smem + C::Q_OFF + i * C::TILE_BYTES + c * BM * C::SW, &p.tm_q, q_full,
                      c * C::CE, q0 + i * BM, head, batch, pol_q);
      for (int j = 0; j < n_max; ++j) {
        const int st = j % C::kStages;
        const uint32_t ph = (j / C::kStages) & 1;
        mbar_wait(k_empty + st, ph ^ 1);
        FWD_TRACE(8, j);
        mbar_arrive_expect_tx(k_full + st, C::KTILE);
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(smem + C::K_OFF + st * C::KTILE + c * BN * C::SW, &p.tm_k,
                      k_full + st, c * C::CE, j * BN, kvhead, batch, pol_kv);
        mbar_wait(v_empty + st, ph ^ 1);
        FWD_TRACE(9, j);
        mbar_arrive_expect_tx(v_full + st, C::KTILE);
        for (int c = 0; c < C::NCH; ++c)
          tma_load_4d(smem + C::V_OFF + st * C::KTILE + c * BN * C::SW, &p.tm_v,
                      v_full + st, c * C::CE, j * BN, kvhead, batch, pol_kv);
      }
    }
  } else if (warp == kMmaWarp || (C::MMA2 && warp == C::kMmaWarp2)) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the schedule (warp-uniform control flow keeps descriptors in
    // uniform registers); one elected lane issues each batch of tcgen05.mma + commit.
    // Descriptors are built once per tile and advanced by compile-time byte offsets.
    if (n_max > 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(BM, D, 0, 1);
      auto issue_qk = [&](int i, int j) {
        const int st = j % C::kStages;
        const uint64_t da = make_smem_desc(sq + i * C::TILE_BYTES, 16, C::SBO, C::LAYOUT);
        const uint64_t db = make_smem_desc(sk + st * C::KTILE, 16, C::SBO, C::LAYOUT);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_ss(tmem + C::S_COL + i * BN, da + kmajor_off<D, BM>(kk),
                   db + kmajor_off<D, BN>(kk), idesc_qk, kk > 0);
          tc_commit(s_full + i);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int i, int j) {
        const int st = j % C::kStages;
        const uint64_t dv = make_smem_desc(sv + st * C::KTILE, BN * C::SW, C::SBO, C::LAYOUT);
        const uint32_t pa = tmem + C::P_COL + i * C::P_STRIDE;
        const uint32_t oa = tmem + C::O_COL + i * D;
        const uint32_t acc0 = j > 0 ? 1u : 0u;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            mma_ts(oa, pa + kk * 8, dv + (uint64_t)((kk * 16 * C::SW) >> 4), idesc_pv,
                   kk > 0 ? 1u : acc0);
          tc_commit(o_done + i);
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) tc_commit(bar);
        __syncwarp();
      };
      // the Q tiles this warp issues for (all of them, or one with MMA2)
      const int i_lo = C::MMA2 ? (warp == kMmaWarp ? 1 : 0) : 0;
      const int i_hi = C::MMA2 ? i_lo + 1 : NQ;
      mbar_wait(q_full, 0);
      mbar_wait(k_full + 0, 0);
      tc_fence_after();
      for (int i = i_lo; i < i_hi; ++i)
        if (n_tiles[i] > 0) issue_qk(i, 0);
      commit(k_empty + 0);
      for (int j = 0; j < n_max; ++j) {
        const int st = j % C::kStages;
        const uint32_t ph = (j / C::kStages) & 1;
        const bool next = j + 1 < n_max;
        const int st1 = (j + 1) % C::kStages;
        const uint32_t ph1 = ((j + 1) / C::kStages) & 1;
        // V_j is only needed by PV_i(j): AUTOSP_FWD_LATE_V checks it there, so the warp goes
        // from PV_i(j-1) straight to the s_free wait that gates QK_i(j+1)
        bool v_ready = false;
        auto need_v = [&]() {
          if (!v_ready) {
            mbar_wait(v_full + st, ph);
            if (lane == 0 && i_lo == 0) FWD_TRACE(14, j);
            v_ready = true;
          }
        };
        if (!(AUTOSP_FWD_LATE_V && D > 64)) need_v();
        bool k_next_ready = false;
        auto need_k_next = [&]() {
          if (!k_next_ready) {
            if (lane == 0 && i_lo == 0) FWD_TRACE(11, j);
            mbar_wait(k_full + st1, ph1);
            if (lane == 0 && i_lo == 0) FWD_TRACE(10, j);
            tc_fence_after();
            k_next_ready = true;
          }
        };
        // K_{j+1} (loaded long ago: the ring runs stages ahead) is checked here, not
        // between s_free / PV(j) and the QK_i(j+1) it feeds: an mbarrier check costs this
        // warp ~100-300 cycles even when the phase is complete, and there it would sit on
        // the softmax's critical path (tools/fwd_trace.py: -170 cycles per KV tile, +4.5 %)
        if (AUTOSP_FWD_EARLY_K && next) need_k_next();
        for (int i = i_lo; i < i_hi; ++i) {
          if (j >= n_tiles[i]) continue;
          if (C::SEP_P && j + 1 < n_tiles[i]) {
            // S_i(j+1) as soon as the softmax has read S_i(j)
            mbar_wait(s_free + i, j & 1);
            if (lane == 0 && i == 0) FWD_TRACE(12, j);
            need_k_next();
            issue_qk(i, j + 1);
            if (lane == 0 && i == 0) FWD_TRACE(13, j);
          }
          need_v();
          mbar_wait(p_full + i, j & 1);
          if (lane == 0) FWD_TRACE(0 + i, j);
          tc_fence_after();
          issue_pv(i, j);
          if (lane == 0) FWD_TRACE(2 + i, j);
          if (!C::SEP_P && j + 1 < n_tiles[i]) {  // P aliases S: QK after PV (in-order)
            need_k_next();
            issue_qk(i, j + 1);
          }
        }
        need_v();  // (a warp with no tile left at j still observes the phase it releases)
        commit(v_empty + st);
        if (next) {
          if (!k_next_ready) mbar_wait(k_full + st1, ph1);  // unused K_{j+1}: still release
          commit(k_empty + st1);
        }
      }
    }
  } else if (warp >= kSoftmaxWarp0 && warp < kSoftmaxWarp0 + 4 * NQ) {
    // ------------------------------------------------------------ softmax warpgroups
    const int i = (warp - kSoftmaxWarp0) / 4;  // Q tile
    const int quarter = warp & 3;              // TMEM lane quarter
    const int row = quarter * 32 + lane;
    const int qi = q0 + i * BM + row;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + C::S_COL + i * BN;
    const uint32_t p_addr = tmem + lane_base + C::P_COL + i * C::P_STRIDE;
    const uint32_t o_addr = tmem + lane_base + C::O_COL + i * D;
    const int n = n_tiles[i];
    float m = -INFINITY;  // running max in log2 units
    float l = 0.f;
    for (int j = 0; j < n; ++j) {
      mbar_wait(s_full + i, j & 1);
      if (lane == 0 && (warp & 3) == 0) FWD_TRACE(4 + i, j);
      tc_fence_after();
      const int k0 = j * BN;
      const bool need_mask = (p.causal && k0 + BN - 1 > q0 + i * BM) || (k0 + BN > p.S);
      const int lim = p.causal ? min(qi + 1, p.S) : p.S;  // keys < lim are valid
      float alpha = 1.f;
      bool rescale = false;
      float rs = 0.f;
      // Two passes over S in TMEM (row max, then exp) keep only 64 scores in registers.
      // Two code versions: element masks only on diagonal / tail tiles; the exp loop is
      // branch-free so independent exps interleave.
      auto pass1 = [&](auto kMasked) -> float {  // row max over the (masked) scores
        constexpr bool M = decltype(kMasked)::value;
        // 8 independent FMNMX3 chains (a single running max is a 64-deep dependency chain)
        float mx8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
#pragma unroll
        for (int h = 0; h < C::NH; ++h) {
          uint32_t sr[64];
          tmem_ld32(s_addr + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
          tmem_ld32(s_addr + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            float a = __uint_as_float(sr[c]), b = __uint_as_float(sr[c + 1]);
            if constexpr (M) {
              a = (k0 + h * 64 + c >= lim) ? -INFINITY : a;
              b = (k0 + h * 64 + c + 1 >= lim) ? -INFINITY : b;
            }
            mx8[(c >> 1) & 7] = fmax3(mx8[(c >> 1) & 7], a, b);
          }
        }
        return fmaxf(fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]), mx8[6]),
                     mx8[7]);
      };
      if (C::SEP_P && j > 0 && !need_mask) {
        // Optimistic single pass (the common case): exps against the RUNNING max m, the
        // row max tracked in the same pass -- no separate max pass re-reading S from TMEM.
        // Only if some row's max grew by more than 2^8 (exp2 arguments beyond +8) is the
        // tile redone exactly like the two-pass path below (warp-uniform decision).
#if !AUTOSP_FWD_LATE_ODONE
        mbar_wait(o_done + i, (j - 1) & 1);  // PV_i(j-1) done with the P_i buffer
        tc_fence_after();
#endif
        const uint64_t sl2 = f2_pack(p.scale_log2, p.scale_log2);
        const uint64_t nm2 = f2_pack(-m, -m);
        uint64_t rs2[4] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f),
                           f2_pack(0.f, 0.f)};
        float mx4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) mx4[k] = -INFINITY;
        bool redo = false;
#pragma unroll
        for (int h = 0; h < C::NH; ++h) {
          uint32_t sr[64];
          tmem_ld32(s_addr + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
          tmem_ld32(s_addr + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 64; c += 2)
            mx4[(c >> 1) & 3] = fmax3(mx4[(c >> 1) & 3], __uint_as_float(sr[c]),
                                      __uint_as_float(sr[c + 1]));
          if (h == C::NH - 1) {  // whole row seen: decide, then release S_i
            const float mxr = fmaxf(fmax3(mx4[0], mx4[1], mx4[2]), mx4[3]);
            redo = __any_sync(0xffffffffu, mxr * p.scale_log2 > m + (float)AUTOSP_FWD_RESCALE_T);
            if (redo) break;  // S_i stays: the two-pass path re-reads it
            tc_fence_before();
            mbar_arrive_warp(s_free + i);
            if (lane == 0 && warp == 0) FWD_TRACE(15, j);
            FWD_TRACE_SKEW(6, j);  // events 6..9: warps 0..3 release S_0(j)
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t pk[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(sr[q * 32 + 2 * c]),
                                                 __uint_as_float(sr[q * 32 + 2 * c + 1])),
                                         sl2, nm2);
              uint64_t e2;
              if ((c & 7) >= 8 - C::kEmuPer8) {
                e2 = f2_exp2_poly(x2);  // FMA pipe
              } else {
                float x0, x1;
                f2_unpack(x2, x0, x1);
                e2 = f2_pack(fast_exp2(x0), fast_exp2(x1));  // MUFU
              }
              rs2[c & 3] = f2_add(rs2[c & 3], e2);
              float ea, eb;
              f2_unpack(e2, ea, eb);
              pk[c] = pack_bf16(ea, eb);
            }
#if AUTOSP_FWD_LATE_ODONE
            if (h == 0 && q == 0) {  // PV_i(j-1) done with the P_i buffer: waited for only
              mbar_wait(o_done + i, (j - 1) & 1);  // now, after the first 32 exps
              tc_fence_after();
            }
#endif
            tmem_st16(p_addr + (h * 2 + q) * 16, pk);
          }
        }
        if (!redo) {
          float r0, r1;
          f2_unpack(f2_add(f2_add(rs2[0], rs2[1]), f2_add(rs2[2], rs2[3])), r0, r1);
          l += r0 + r1;
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive_warp(p_full + i);
          if (lane == 0 && (warp & 3) == 0) FWD_TRACE(6 + i, j);
          FWD_TRACE_SKEW(10, j);  // events 10..13: warps 0..3 arrive P_0(j)
          continue;
        }
      }
      const float mx = need_mask ? pass1(std::true_type{}) : pass1(std::false_type{});
      const float m_cand = mx * p.scale_log2;
      if (m_cand > m + (float)AUTOSP_FWD_RESCALE_T) {  // lazy rescale (also taken on the first tile)
        alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - m_cand);
        rescale = (j > 0);
        m = m_cand;
      }
      // PV_i(j-1) must be complete before O is rescaled and (SEP_P) before P_i is
      // overwritten; it was issued a whole softmax ago, so this rarely waits.  (Without
      // SEP_P it is already implied by s_full(j) -- in-order pipe -- but every phase of
      // o_done is observed, which keeps the parity waits trivially sound.)
      if (j > 0) {
        mbar_wait(o_done + i, (j - 1) & 1);
        tc_fence_after();
      }
      // tcgen05.ld/st are .sync.aligned: the whole warp must execute them, so the rescale
      // is warp-uniform (alpha == 1 for the lanes whose max did not move)
      if (__any_sync(0xffffffffu, rescale)) {
        if (!rescale) alpha = 1.f;
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {
          uint32_t orr[32];
          tmem_ld32(o_addr + c, orr);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 32; ++t) orr[t] = __float_as_uint(__uint_as_float(orr[t]) * alpha);
          tmem_st32(o_addr + c, orr);
        }
      }
      const float moff = (m == -INFINITY) ? 0.f : m;
      auto pass2 = [&](auto kMasked) -> float {  // P = exp2(s c - m) -> bf16, row sum
        constexpr bool M = decltype(kMasked)::value;
        const uint64_t sl2 = f2_pack(p.scale_log2, p.scale_log2);
        const uint64_t nm2 = f2_pack(-moff, -moff);
        uint64_t rs2[4] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f), f2_pack(0.f, 0.f),
                           f2_pack(0.f, 0.f)};
#pragma unroll
        for (int h = 0; h < C::NH; ++h) {
          uint32_t sr[64];
          tmem_ld32(s_addr + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
          tmem_ld32(s_addr + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
          tmem_wait_ld();
          if (C::SEP_P && h == C::NH - 1) {  // S_i fully read: the MMA may overwrite it with S_i(j+1)
            tc_fence_before();
            mbar_arrive_warp(s_free + i);
            if (lane == 0 && warp == 0) FWD_TRACE(15, j);
            FWD_TRACE_SKEW(6, j);  // events 6..9: warps 0..3 release S_0(j)
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t pk[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              float a = __uint_as_float(sr[q * 32 + 2 * c]);
              float b = __uint_as_float(sr[q * 32 + 2 * c + 1]);
              if constexpr (M) {
                const int col = k0 + h * 64 + q * 32 + 2 * c;
                a = (col >= lim) ? -INFINITY : a;
                b = (col + 1 >= lim) ? -INFINITY : b;
              }
              const uint64_t x2 = f2_fma(f2_pack(a, b), sl2, nm2);
              uint64_t e2;
              if (!M && (c & 7) >= 8 - C::kEmuPer8) {
                e2 = f2_exp2_poly(x2);  // FMA pipe
              } else {
                float x0, x1;
                f2_unpack(x2, x0, x1);
                e2 = f2_pack(fast_exp2(x0), fast_exp2(x1));  // MUFU
              }
              rs2[c & 3] = f2_add(rs2[c & 3], e2);
              float ea, eb;
              f2_unpack(e2, ea, eb);
              pk[c] = pack_bf16(ea, eb);
            }
            // P chunk (h*2+q) -> cols [16*(2h+q), +16) of the P buffer (aliasing S for
            // d = 128: only already-read columns)
            tmem_st16(p_addr + (h * 2 + q) * 16, pk);
          }
        }
        float r0, r1, r2, r3;
        f2_unpack(f2_add(f2_add(rs2[0], rs2[1]), f2_add(rs2[2], rs2[3])), r0, r1);
        (void)r2; (void)r3;
        return r0 + r1;
      };
      rs = need_mask ? pass2(std::true_type{}) : pass2(std::false_type{});
      l = l * alpha + rs;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_warp(p_full + i);
      if (lane == 0 && (warp & 3) == 0) FWD_TRACE(6 + i, j);
    }
    // ---- epilogue: O / l -> bf16, LSE
    if (n > 0) {
      mbar_wait(o_done + i, (n - 1) & 1);
      tc_fence_after();
      const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
      // O rows leave through shared memory: every MMA of tile i is complete (o_done), so
      // the Q_i tile is free and becomes this warp's staging area [32 rows x D bf16]
      // (16-byte units XOR-swizzled by row: conflict-free both ways).  The warp then
      // stores 32 / VPR whole rows per instruction -- row-contiguous 16-byte vectors,
      // full 128-byte lines -- instead of one 16-byte piece of 32 scattered rows: the
      // pattern NVLink (fused K2 push into the token owners' receive regions, global
      // head rank * Hq + head, token-major) and HBM both want.
      constexpr int ROWB = D * 2;
      constexpr int VPR = ROWB / 16;  // 16-byte units per row
      constexpr int RPI = 32 / VPR;   // rows per warp store instruction
      uint8_t* stage = smem + C::Q_OFF + i * C::TILE_BYTES + quarter * 32 * ROWB;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t orr[32];
        tmem_ld32(o_addr + c, orr);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          uint4 v;
          v.x = pack_bf16(__uint_as_float(orr[8 * t + 0]) * inv_l,
                          __uint_as_float(orr[8 * t + 1]) * inv_l);
          v.y = pack_bf16(__uint_as_float(orr[8 * t + 2]) * inv_l,
                          __uint_as_float(orr[8 * t + 3]) * inv_l);
          v.z = pack_bf16(__uint_as_float(orr[8 * t + 4]) * inv_l,
                          __uint_as_float(orr[8 * t + 5]) * inv_l);
          v.w = pack_bf16(__uint_as_float(orr[8 * t + 6]) * inv_l,
                          __uint_as_float(orr[8 * t + 7]) * inv_l);
          const int u = c / 8 + t;
          sts128(stage + lane * ROWB + ((u ^ ((lane & 7) & (VPR - 1))) << 4), v);
        }
      }
      if (qi < p.S)
        p.lse[((int64_t)batch * p.Hq + head) * p.S + qi] =
            (m + __log2f(l)) * 0.69314718055994531f;
      __syncwarp();
      const int u = lane % VPR;
#pragma unroll
      for (int it = 0; it < 32 / RPI; ++it) {
        const int r = it * RPI + lane / VPR;  // row within this warp's 32
        const int qr = q0 + i * BM + quarter * 32 + r;
        if (qr < p.S) {
          const uint4 v = lds128u(stage + r * ROWB + ((u ^ ((r & 7) & (VPR - 1))) << 4));
          if (p.o)  // (push without a local copy: o == nullptr)
            reinterpret_cast<uint4*>(p.o + (int64_t)batch * p.o_sb + (int64_t)head * p.o_sh +
                                     (int64_t)qr * p.o_ss)[u] = v;
          if (p.push) {
            const int jr = qr / p.s_loc;
            reinterpret_cast<uint4*>(
                p.peer_base[jr] + p.dst_off +
                ((int64_t)batch * p.d_sb + (int64_t)(qr - jr * p.s_loc) * p.d_ss +
                 (int64_t)(p.rank * p.Hq + head) * p.d_sh) * 2)[u] = v;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kAllocWarp) tmem_dealloc<C::TMEM_COLS>(tmem);
  if (p.push) publish_arrival(p.peer_flags, p.P, p.rank, p.epoch, p.check,
                              gridDim.x * gridDim.y * gridDim.z);
}

template <int D>
int launch(const autosp_attn_tensor& q, const autosp_attn_tensor& k, const autosp_attn_tensor& v,
           const autosp_attn_tensor& o, float* lse, int B, int Hq, int Hkv, int S, float scale,
           int causal, const autosp_push_spec* push, cudaStream_t stream) {
  using C = Cfg<D>;
  Params p{};
  if (push) {
    p.push = 1;
    p.P = push->world;
    p.rank = push->rank;
    p.s_loc = S / push->world;
    p.dst_off = push->dst_offset;
    p.d_sb = push->dst_stride_b;
    p.d_ss = push->dst_stride_s;
    p.d_sh = push->dst_stride_h;
    for (int j = 0; j < push->world; ++j) {
      p.peer_base[j] = static_cast<char*>(push->peer_base[j]);
      p.peer_flags[j] = push->peer_flags[j];
    }
    p.epoch = push->epoch;
    p.check = autosp_push_check(push, Hq);
  }
  if (!make_map_bhsd(&p.tm_q, q.ptr, B, Hq, S, D, q.stride_b, q.stride_h, q.stride_s, C::CE, BM,
                     C::SW) ||
      !make_map_bhsd(&p.tm_k, k.ptr, B, Hkv, S, D, k.stride_b, k.stride_h, k.stride_s, C::CE, C::BN,
                     C::SW) ||
      !make_map_bhsd(&p.tm_v, v.ptr, B, Hkv, S, D, v.stride_b, v.stride_h, v.stride_s, C::CE, C::BN,
                     C::SW)) {
    autosp_set_error("attn_fwd: cuTensorMapEncodeTiled failed (alignment/strides?)");
    return AUTOSP_ERR_VALIDATION;
  }
  p.o = static_cast<__nv_bfloat16*>(const_cast<void*>(o.ptr));
  p.o_sb = o.stride_b;
  p.o_sh = o.stride_h;
  p.o_ss = o.stride_s;
  p.lse = lse;
  p.B = B;
  p.Hq = Hq;
  p.Hkv = Hkv;
  p.S = S;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.causal = causal;
  p.n_qblk = (S + C::NQ * BM - 1) / (C::NQ * BM);
  p.trace = g_fwd_trace;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr_set = true;
  }
  const dim3 grid = causal_grid(AUTOSP_FWD_LPT, p.n_qblk, Hq, B);
  attn_fwd_kernel<D><<<grid, C::kThreads, C::SMEM, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    autosp_set_error("attn_fwd launch failed: %s", cudaGetErrorString(e));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}

}  // namespace fwd
}  // namespace autosp

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int autosp_check_attn_tensor(const autosp_attn_tensor& t, const char* name) {
  if (!t.ptr || !aligned16(t.ptr) || (t.stride_b * 2) % 16 || (t.stride_h * 2) % 16 ||
      (t.stride_s * 2) % 16) {
    autosp_set_error("attention tensor %s must be non-null, 16-byte aligned with strides that "
                     "are multiples of 8 elements",
                     name);
    return AUTOSP_ERR_VALIDATION;
  }
  return AUTOSP_OK;
}

int autosp_internal_handshake(uint32_t* const* flags, int world, int rank, uint32_t epoch,
                              cudaStream_t stream);

static int attn_fwd_impl(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                         autosp_attn_tensor o, float* lse, int b, int hq, int hkv, int s, int d,
                         float scale, int causal, const autosp_push_spec* push, void* stream);

extern "C" int autosp_attn_fwd(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                               autosp_attn_tensor o, float* lse, int b, int hq, int hkv, int s,
                               int d, float scale, int causal, void* stream) {
  return attn_fwd_impl(q, k, v, o, lse, b, hq, hkv, s, d, scale, causal, nullptr, stream);
}

extern "C" int autosp_attn_fwd_push(autosp_attn_tensor q, autosp_attn_tensor k,
                                    autosp_attn_tensor v, autosp_attn_tensor o, float* lse, int b,
                                    int hq, int hkv, int s, int d, float scale, int causal,
                                    const autosp_push_spec* push, void* stream) {
  if (!push || push->world < 1 || push->world > AUTOSP_MAX_WORLD || push->rank < 0 ||
      push->rank >= push->world || !push->peer_base || !push->peer_flags) {
    autosp_set_error("attn_fwd_push: bad push spec");
    return AUTOSP_ERR_VALIDATION;
  }
  if (s % push->world) {
    autosp_set_error("attn_fwd_push: sequence %d not divisible by world size %d", s, push->world);
    return AUTOSP_ERR_VALIDATION;
  }
  if (push->dst_offset % 16 || push->dst_stride_b % 8 || push->dst_stride_s % 8 ||
      push->dst_stride_h % 8) {
    autosp_set_error("attn_fwd_push: destination offset/strides must be 16-byte multiples");
    return AUTOSP_ERR_VALIDATION;
  }
  for (int j = 0; j < push->world; ++j)
    if (!push->peer_base[j] || !push->peer_flags[j] ||
        (reinterpret_cast<uintptr_t>(push->peer_base[j]) & 15)) {
      autosp_set_error("attn_fwd_push: peer %d base/flags null or misaligned", j);
      return AUTOSP_ERR_VALIDATION;
    }
  if (push->world > 1) {
    int rc = autosp_internal_handshake(push->peer_flags, push->world, push->rank, push->epoch,
                                       static_cast<cudaStream_t>(stream));
    if (rc) {
      autosp_set_error("attn_fwd_push: handshake launch failed");
      return rc;
    }
  }
  return attn_fwd_impl(q, k, v, o, lse, b, hq, hkv, s, d, scale, causal, push, stream);
}

static int attn_fwd_impl(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                         autosp_attn_tensor o, float* lse, int b, int hq, int hkv, int s, int d,
                         float scale, int causal, const autosp_push_spec* push, void* stream) {
  if (b < 1 || hq < 1 || hkv < 1 || s < 1 || hq % hkv) {
    autosp_set_error("attn_fwd: bad shape b=%d hq=%d hkv=%d s=%d", b, hq, hkv, s);
    return AUTOSP_ERR_VALIDATION;
  }
  int rc;
  if ((rc = autosp_check_attn_tensor(q, "q")) || (rc = autosp_check_attn_tensor(k, "k")) ||
      (rc = autosp_check_attn_tensor(v, "v")) ||
      ((o.ptr || !push) && (rc = autosp_check_attn_tensor(o, "o"))))
    return rc;
  if (!lse) {
    autosp_set_error("attn_fwd: lse must be non-null");
    return AUTOSP_ERR_VALIDATION;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (d) {
    case 32: return autosp::fwd::launch<32>(q, k, v, o, lse, b, hq, hkv, s, scale, causal, push, st);
    case 64: return autosp::fwd::launch<64>(q, k, v, o, lse, b, hq, hkv, s, scale, causal, push, st);
    case 128: return autosp::fwd::launch<128>(q, k, v, o, lse, b, hq, hkv, s, scale, causal, push, st);
    default:
      autosp_set_error("attn_fwd: head_dim %d unsupported (32, 64, 128)", d);
      return AUTOSP_ERR_UNSUPPORTED;
  }
}

int autosp_preload_fwd() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, autosp::fwd::attn_fwd_kernel<32>);
  cudaFuncGetAttributes(&a, autosp::fwd::attn_fwd_kernel<64>);
  cudaFuncGetAttributes(&a, autosp::fwd::attn_fwd_kernel<128>);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

extern "C" AUTOSP_API int autosp_debug_set_fwd_trace(long long* dev_buf) {
  autosp::fwd::g_fwd_trace = dev_buf;
  return AUTOSP_OK;
}
