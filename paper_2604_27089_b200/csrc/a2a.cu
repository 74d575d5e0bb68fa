// K1 / K2: the Ulysses all-to-all reshard as ONE push kernel over NVLink/NVSwitch peer
// memory.  Semantics = all_to_all_shards (reference executor.py:203-230): a pure index
// permutation, so the result is bit-exact.
//
// Design (B200):
//  * every rank PUSHES its slabs straight into each peer's symmetric receive region
//    (mapped once via CUDA IPC) with 16-byte vector stores; no staging, no NCCL;
//  * source/destination are arbitrary (b, s, h) strided views with head_dim contiguous,
//    so the QKV-projection output [b, s/P, (hq+2hkv)*d] is read in place and written as
//    the head-major [b, h/P, s, d] attention operand (the transpose is folded in), and
//    the attention output is written back as the token-major O-projection input;
//  * a warp owns (tensor, batch, head, 16-token tile): source rows are 128B-line
//    coalesced, destination rows of consecutive tokens are contiguous, loads are issued
//    in a batch before the stores (latency of remote HBM is hidden by MLP);
//  * cross-GPU ordering with two epoch flags per rank and no host synchronisation:
//    "ready" (I have reached call e: my readers of older data are stream-ordered
//    before me) and "arrive[src]" (src finished writing call e into me).  All spins are
//    bounded by %globaltimer and trap instead of hanging the GPU.
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/autosp.h"
#include <cuda_bf16.h>

#include "flags.cuh"
#include "ptx.cuh"
#include "rope.cuh"

namespace autosp {
#ifndef AUTOSP_A2A_BPS
#define AUTOSP_A2A_BPS 4  // push CTAs per SM (grid cap; A/B: 1, 2, 8, 16 slower)
#endif
#ifndef AUTOSP_A2A_TILE
#define AUTOSP_A2A_TILE 16  // tokens per warp item of the push kernels
#endif
constexpr int kTileTokens = AUTOSP_A2A_TILE;
constexpr int kA2AThreads = 256;

struct A2ATensorDev {
  const char* src;
  int64_t ss_b, ss_s, ss_h;  // element strides
  int64_t dst_off;           // bytes
  int64_t ds_b, ds_s, ds_h;  // element strides
  int heads;
  int tiles;                 // token tiles of the source
  int64_t items;             // b * heads * tiles
  int rope;                  // 1: apply RoPE (bf16 rows) at the source token's position
};

struct A2AParams {
  A2ATensorDev t[AUTOSP_A2A_MAX_TENSORS];
  int n;
  int dir;
  int b, s_loc, s_glob, d, eb;
  int P, rank;
  char* peer_base[AUTOSP_MAX_WORLD];
  uint32_t* peer_flags[AUTOSP_MAX_WORLD];
  uint32_t epoch;
  uint32_t check;
  int64_t total_items;
  const float* pos;  // RoPE positions of the SOURCE tokens (seq_to_head: the local shard)
  float log2_theta;
  uint64_t timeout_ns;  // flag spins trap after this long (autosp_set_spin_timeout)
};

AUTOSP_DEV bool epoch_reached(uint32_t v, uint32_t e) { return (int32_t)(v - e) >= 0; }

AUTOSP_DEV void spin_until_epoch(const uint32_t* p, uint32_t e, uint64_t timeout_ns) {
  if (epoch_reached(ld_acquire_sys(p), e)) return;
  uint64_t t0 = globaltimer();
  while (!epoch_reached(ld_acquire_sys(p), e)) {
    if (globaltimer() - t0 > timeout_ns) {
      printf("autosp: peer flag wait timed out after %llu ns (epoch %u, flag %u)\n",
             (unsigned long long)timeout_ns, e, ld_acquire_sys(p));
      asm volatile("trap;");
    }
    __nanosleep(64);
  }
}

AUTOSP_DEV void push_complete(const A2AParams& p) {
  publish_arrival(p.peer_flags, p.P, p.rank, p.epoch, p.check, gridDim.x);
}

// Fast path: 16-byte vectors, rows of ROWB = d * elem_bytes in {64, 128, 256} bytes.  A
// warp owns (tensor, batch, head, 16-token tile); everything but the token offset is
// hoisted out of the row loop (the generic kernel below recomputed 64-bit strided
// addresses and integer divisions for all 16 possible row passes, predicated, and was
// instruction-bound at ~0.5 TB/s).
AUTOSP_DEV float p_pos(const float* pos, int t) { return __ldg(pos + t); }

template <int ROWB>
__global__ void __launch_bounds__(kA2AThreads) a2a_push_fast(const __grid_constant__ A2AParams p) {
  constexpr int VPR = ROWB / 16;          // vectors per row
  constexpr int RPP = 32 / VPR;           // rows per pass
  constexpr int PASSES = kTileTokens / RPP;
  const int lane = threadIdx.x & 31;
  const int r_in = lane / VPR;
  const int voff = (lane % VPR) * 16;
  const bool s2h = p.dir == AUTOSP_SEQ_TO_HEAD;
  const int s_src = s2h ? p.s_loc : p.s_glob;
  const int warps_total = gridDim.x * (kA2AThreads / 32);
  const int gw = blockIdx.x * (kA2AThreads / 32) + (threadIdx.x >> 5);
  const int total = (int)p.total_items;
  for (int item = gw; item < total; item += warps_total) {
    int it = item;
    const A2ATensorDev* T = &p.t[0];
#pragma unroll
    for (int k = 1; k < AUTOSP_A2A_MAX_TENSORS; ++k)
      if (k < p.n && it >= (int)T->items) { it -= (int)T->items; T = &p.t[k]; }
    const int tile = it % T->tiles;
    const int bh = it / T->tiles;
    const int hh = bh % T->heads;
    const int bi = bh / T->heads;
    const int t0 = tile * kTileTokens;
    const int eb = p.eb;
    const char* src = T->src + ((int64_t)bi * T->ss_b + (int64_t)t0 * T->ss_s +
                                (int64_t)hh * T->ss_h) * eb + voff;
    const int64_t sstep = T->ss_s * eb;
    const int64_t dstep = T->ds_s * eb;
    const int last = min(t0 + kTileTokens, s_src) - 1;
    uint4 v[PASSES];
#pragma unroll
    for (int ps = 0; ps < PASSES; ++ps) {
      const int r = ps * RPP + r_in;
      if (t0 + r <= last) v[ps] = __ldg(reinterpret_cast<const uint4*>(src + r * sstep));
    }
    if (T->rope) {
      // RoPE folded into the reshard (bf16 rows): the rotation partner of this lane's 8
      // elements is the lane holding the other half of the row (lane ^ VPR/2, same row)
      const int vin = lane % VPR;
      const bool hi = vin >= VPR / 2;
      const int d = ROWB / 2;
#pragma unroll
      for (int ps = 0; ps < PASSES; ++ps) {
        const int r = ps * RPP + r_in;
        uint4 o;
        o.x = __shfl_xor_sync(0xffffffffu, v[ps].x, VPR / 2);
        o.y = __shfl_xor_sync(0xffffffffu, v[ps].y, VPR / 2);
        o.z = __shfl_xor_sync(0xffffffffu, v[ps].z, VPR / 2);
        o.w = __shfl_xor_sync(0xffffffffu, v[ps].w, VPR / 2);
        if (t0 + r <= last) {
          const float tp = p_pos(p.pos, t0 + r);
          const __nv_bfloat162* mine = reinterpret_cast<const __nv_bfloat162*>(&v[ps]);
          const __nv_bfloat162* other = reinterpret_cast<const __nv_bfloat162*>(&o);
          uint4 res;
          __nv_bfloat162* out = reinterpret_cast<__nv_bfloat162*>(&res);
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            const float2 m2 = __bfloat1622float2(mine[k2]);
            const float2 o2 = __bfloat1622float2(other[k2]);
            float s0, c0, s1, c1;
            const int j0 = (vin % (VPR / 2)) * 8 + 2 * k2;
            rope_sincos(tp, j0, d, p.log2_theta, &s0, &c0);
            rope_sincos(tp, j0 + 1, d, p.log2_theta, &s1, &c1);
            const float y0 = hi ? rope_hi(o2.x, m2.x, c0, s0) : rope_lo(m2.x, o2.x, c0, s0);
            const float y1 = hi ? rope_hi(o2.y, m2.y, c1, s1) : rope_lo(m2.y, o2.y, c1, s1);
            out[k2] = __floats2bfloat162_rn(y0, y1);
          }
          v[ps] = res;
        }
      }
    }
    if (s2h) {
      const int hl = T->heads / p.P;
      const int j = hh / hl;
      char* dst = p.peer_base[j] + T->dst_off +
                  ((int64_t)bi * T->ds_b + (int64_t)(p.rank * p.s_loc + t0) * T->ds_s +
                   (int64_t)(hh - j * hl) * T->ds_h) * eb + voff;
#pragma unroll
      for (int ps = 0; ps < PASSES; ++ps) {
        const int r = ps * RPP + r_in;
        if (t0 + r <= last) *reinterpret_cast<uint4*>(dst + r * dstep) = v[ps];
      }
    } else {
      const int dh = p.rank * T->heads + hh;
      const int j0 = t0 / p.s_loc;
      if (last / p.s_loc == j0) {  // tile inside one destination rank's token range
        char* dst = p.peer_base[j0] + T->dst_off +
                    ((int64_t)bi * T->ds_b + (int64_t)(t0 - j0 * p.s_loc) * T->ds_s +
                     (int64_t)dh * T->ds_h) * eb + voff;
#pragma unroll
        for (int ps = 0; ps < PASSES; ++ps) {
          const int r = ps * RPP + r_in;
          if (t0 + r <= last) *reinterpret_cast<uint4*>(dst + r * dstep) = v[ps];
        }
      } else {
#pragma unroll
        for (int ps = 0; ps < PASSES; ++ps) {
          const int t = t0 + ps * RPP + r_in;
          if (t <= last) {
            const int j = t / p.s_loc;
            char* dst = p.peer_base[j] + T->dst_off +
                        ((int64_t)bi * T->ds_b + (int64_t)(t - j * p.s_loc) * T->ds_s +
                         (int64_t)dh * T->ds_h) * eb + voff;
            *reinterpret_cast<uint4*>(dst) = v[ps];
          }
        }
      }
    }
  }
  push_complete(p);
}

// The backward's seq->head reshard of the attention-output gradient, fused with
// delta = rowsum(dO * O) (the softmax-gradient correction term, reference softmax_dx
// executor.py:89-91, formed on the token owner where O lives): tensor 0 of the call is
// dO (pushed head-major like any a2a tensor), tensor 1 describes O (its source) and the
// fp32 delta destination [b, h/P, S].  One warp per (batch, head, 16-token tile); the
// row's lanes reduce their 8-element partial dot products with shuffles.
template <int ROWB>
__global__ void __launch_bounds__(kA2AThreads) a2a_grad_out_kernel(const __grid_constant__ A2AParams p) {
  constexpr int VPR = ROWB / 16;
  constexpr int RPP = 32 / VPR;
  constexpr int PASSES = kTileTokens / RPP;
  const int lane = threadIdx.x & 31;
  const int r_in = lane / VPR;
  const int voff = (lane % VPR) * 16;
  const A2ATensorDev& G = p.t[0];
  const A2ATensorDev& O = p.t[1];
  const int warps_total = gridDim.x * (kA2AThreads / 32);
  const int total = (int)G.items;
  for (int item = blockIdx.x * (kA2AThreads / 32) + (threadIdx.x >> 5); item < total;
       item += warps_total) {
    const int tile = item % G.tiles;
    const int bh = item / G.tiles;
    const int hh = bh % G.heads;
    const int bi = bh / G.heads;
    const int t0 = tile * kTileTokens;
    const int last = min(t0 + kTileTokens, p.s_loc) - 1;
    const char* gsrc = G.src + ((int64_t)bi * G.ss_b + (int64_t)t0 * G.ss_s +
                                (int64_t)hh * G.ss_h) * 2 + voff;
    const char* osrc = O.src + ((int64_t)bi * O.ss_b + (int64_t)t0 * O.ss_s +
                                (int64_t)hh * O.ss_h) * 2 + voff;
    uint4 g[PASSES], o[PASSES];
#pragma unroll
    for (int ps = 0; ps < PASSES; ++ps) {
      const int r = ps * RPP + r_in;
      if (t0 + r <= last) {
        g[ps] = __ldg(reinterpret_cast<const uint4*>(gsrc + r * G.ss_s * 2));
        o[ps] = __ldg(reinterpret_cast<const uint4*>(osrc + r * O.ss_s * 2));
      }
    }
    const int hl = G.heads / p.P;
    const int j = hh / hl;
    const int64_t tok = (int64_t)p.rank * p.s_loc + t0;
    char* gdst = p.peer_base[j] + G.dst_off +
                 ((int64_t)bi * G.ds_b + tok * G.ds_s + (int64_t)(hh - j * hl) * G.ds_h) * 2 + voff;
    float* ddst = reinterpret_cast<float*>(p.peer_base[j] + O.dst_off) +
                  ((int64_t)bi * O.ds_b + tok * O.ds_s + (int64_t)(hh - j * hl) * O.ds_h);
#pragma unroll
    for (int ps = 0; ps < PASSES; ++ps) {
      const int r = ps * RPP + r_in;
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g[ps]);
      const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&o[ps]);
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 a = __bfloat1622float2(g2[k]), b = __bfloat1622float2(o2[k]);
        acc = fmaf(a.x, b.x, fmaf(a.y, b.y, acc));
      }
#pragma unroll
      for (int off = VPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (t0 + r <= last) {
        *reinterpret_cast<uint4*>(gdst + r * G.ds_s * 2) = g[ps];
        if (lane % VPR == 0) ddst[r * O.ds_s] = acc;
      }
    }
  }
  push_complete(p);
}

// G = bytes moved per lane per row-chunk (16, 8, 4 or 2).
template <typename V>
__global__ void __launch_bounds__(kA2AThreads) a2a_push_kernel(const __grid_constant__ A2AParams p) {
  constexpr int G = sizeof(V);
  const int tid = threadIdx.x;
  // (the ready handshake ran in a2a_handshake_kernel just before, stream-ordered)

  const int vpr = p.d * p.eb / G;  // vectors per row (1..32)
  const int rows_per_pass = min(32 / vpr, kTileTokens);
  const int lane = tid & 31;
  const int r_in_pass = lane / vpr;
  const int v_in_row = lane % vpr;
  const bool lane_active = r_in_pass < rows_per_pass;
  const int warps_total = gridDim.x * (kA2AThreads / 32);
  const int64_t gw = (int64_t)blockIdx.x * (kA2AThreads / 32) + (tid >> 5);

  for (int64_t item = gw; item < p.total_items; item += warps_total) {
    int ti = 0;
    int64_t it = item;
    while (ti < p.n - 1 && it >= p.t[ti].items) { it -= p.t[ti].items; ++ti; }
    const A2ATensorDev& T = p.t[ti];
    const int tile = (int)(it % T.tiles);
    const int64_t bh = it / T.tiles;
    const int hh = (int)(bh % T.heads);
    const int bi = (int)(bh / T.heads);
    const int s_src = (p.dir == AUTOSP_SEQ_TO_HEAD) ? p.s_loc : p.s_glob;
    const int t0 = tile * kTileTokens;
    const int hl = T.heads / p.P;  // seq_to_head: heads per destination rank

    constexpr int kMaxPass = kTileTokens;  // vpr==32 -> 1 row per pass
    V vals[kMaxPass];
    const int passes = (kTileTokens + rows_per_pass - 1) / rows_per_pass;
#pragma unroll
    for (int ps = 0; ps < kMaxPass; ++ps) {
      if (ps < passes) {
        const int t = t0 + ps * rows_per_pass + r_in_pass;
        if (lane_active && t < s_src) {
          const char* src = T.src + ((int64_t)bi * T.ss_b + (int64_t)t * T.ss_s +
                                     (int64_t)hh * T.ss_h) * p.eb;
          vals[ps] = __ldg(reinterpret_cast<const V*>(src) + v_in_row);
        }
      }
    }
#pragma unroll
    for (int ps = 0; ps < kMaxPass; ++ps) {
      if (ps < passes) {
        const int t = t0 + ps * rows_per_pass + r_in_pass;
        if (lane_active && t < s_src) {
          int j, dt, dh;
          if (p.dir == AUTOSP_SEQ_TO_HEAD) {
            j = hh / hl; dt = p.rank * p.s_loc + t; dh = hh - j * hl;
          } else {
            j = t / p.s_loc; dt = t - j * p.s_loc; dh = p.rank * T.heads + hh;
          }
          char* dst = p.peer_base[j] + T.dst_off +
                      ((int64_t)bi * T.ds_b + (int64_t)dt * T.ds_s + (int64_t)dh * T.ds_h) * p.eb;
          reinterpret_cast<V*>(dst)[v_in_row] = vals[ps];
        }
      }
    }
  }

  push_complete(p);
}

// 0) publish "I reached epoch" and wait until every peer has reached it too.  One CTA:
//    the only spinning work of a call is tiny, so it can never starve the push kernels of
//    other ranks sharing the GPU (single-GPU loopback) and costs one short launch.
__global__ void a2a_handshake_kernel(const __grid_constant__ A2AParams p) {
  const int tid = threadIdx.x;
  if (tid == 0) st_release_sys(p.peer_flags[p.rank] + kReadyWord, p.epoch);
  if (tid < p.P && tid != p.rank)
    spin_until_epoch(p.peer_flags[tid] + kReadyWord, p.epoch, p.timeout_ns);
}

struct ShakeParams {
  uint32_t* flags[AUTOSP_MAX_WORLD];
  int P, rank;
  uint32_t epoch;
  uint64_t timeout_ns;
};
__global__ void handshake_kernel(const __grid_constant__ ShakeParams s) {
  const int tid = threadIdx.x;
  if (tid == 0) st_release_sys(s.flags[s.rank] + kReadyWord, s.epoch);
  if (tid < s.P && tid != s.rank) spin_until_epoch(s.flags[tid] + kReadyWord, s.epoch, s.timeout_ns);
}

__global__ void a2a_wait_kernel(uint32_t* flags, int P, int rank, uint32_t epoch,
                                uint32_t check, uint64_t timeout_ns) {
  const int j = threadIdx.x;
  if (j < P && j != rank) {
    spin_until_epoch(flags + kArriveWord + j, epoch, timeout_ns);
    // every sender must have written where this rank expects the data (symmetric
    // allocation invariant); a divergence is a bug -> fail loudly, never corrupt silently
    if (*(volatile uint32_t*)(flags + kCheckWord + j) != check) asm volatile("trap;");
  }
  __syncthreads();
}

struct MarkParams {
  uint32_t* flags[AUTOSP_MAX_WORLD];
  int P;
  uint32_t epoch;
};
__global__ void a2a_mark_ready_kernel(const __grid_constant__ MarkParams m) {
  const int j = threadIdx.x;
  if (j < m.P) st_release_sys(m.flags[j] + kReadyWord, m.epoch);
}

}  // namespace autosp

// ---------------------------------------------------------------------------- C ABI
extern "C" void autosp_set_error(const char* fmt, ...);

// bound of every flag spin (peer ready / arrival); host-side, copied into each launch
static uint64_t g_spin_timeout_ns = 300ull * 1000000000ull;

extern "C" int autosp_set_spin_timeout(double seconds) {
  if (!(seconds > 0.0) || seconds > 1e7) {
    autosp_set_error("spin timeout %g s out of range", seconds);
    return AUTOSP_ERR_VALIDATION;
  }
  g_spin_timeout_ns = (uint64_t)(seconds * 1e9);
  return AUTOSP_OK;
}

static int a2a_impl(int direction, const autosp_a2a_tensor* tensors, int n_tensors, int b,
                    int s_global, int d, int elem_bytes, int world, int rank,
                    void* const* peer_base, uint32_t* const* peer_flags, uint32_t epoch,
                    const float* pos, float theta, void* stream);

extern "C" int autosp_a2a(int direction, const autosp_a2a_tensor* tensors, int n_tensors, int b,
                          int s_global, int d, int elem_bytes, int world, int rank,
                          void* const* peer_base, uint32_t* const* peer_flags, uint32_t epoch,
                          void* stream) {
  for (int i = 0; tensors && i < n_tensors && i < AUTOSP_A2A_MAX_TENSORS; ++i)
    if (tensors[i].rope) {
      autosp_set_error("autosp_a2a: tensor %d requests RoPE; use autosp_a2a_rope", i);
      return AUTOSP_ERR_VALIDATION;
    }
  return a2a_impl(direction, tensors, n_tensors, b, s_global, d, elem_bytes, world, rank,
                  peer_base, peer_flags, epoch, nullptr, 0.f, stream);
}

extern "C" int autosp_a2a_rope(int direction, const autosp_a2a_tensor* tensors, int n_tensors,
                               int b, int s_global, int d, int elem_bytes, int world, int rank,
                               void* const* peer_base, uint32_t* const* peer_flags,
                               uint32_t epoch, const float* pos, float theta, void* stream) {
  if (direction != AUTOSP_SEQ_TO_HEAD || elem_bytes != 2 || !pos || theta <= 1.f ||
      (d != 32 && d != 64 && d != 128)) {
    autosp_set_error("autosp_a2a_rope: seq_to_head of bf16 rows with d in {32, 64, 128}, "
                     "positions and theta > 1 required");
    return AUTOSP_ERR_VALIDATION;
  }
  return a2a_impl(direction, tensors, n_tensors, b, s_global, d, elem_bytes, world, rank,
                  peer_base, peer_flags, epoch, pos, theta, stream);
}

static int a2a_impl(int direction, const autosp_a2a_tensor* tensors, int n_tensors, int b,
                    int s_global, int d, int elem_bytes, int world, int rank,
                    void* const* peer_base, uint32_t* const* peer_flags, uint32_t epoch,
                    const float* pos, float theta, void* stream) {
  using namespace autosp;
  if (direction != AUTOSP_SEQ_TO_HEAD && direction != AUTOSP_HEAD_TO_SEQ) {
    autosp_set_error("unknown all-to-all direction %d", direction);
    return AUTOSP_ERR_VALIDATION;
  }
  if (world < 1 || world > AUTOSP_MAX_WORLD || rank < 0 || rank >= world) {
    autosp_set_error("world %d / rank %d out of range (max world %d)", world, rank,
                     AUTOSP_MAX_WORLD);
    return AUTOSP_ERR_VALIDATION;
  }
  if (n_tensors < 1 || n_tensors > AUTOSP_A2A_MAX_TENSORS || !tensors) {
    autosp_set_error("n_tensors %d out of range", n_tensors);
    return AUTOSP_ERR_VALIDATION;
  }
  if (b < 1 || s_global < 1 || d < 1 || (elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 8)) {
    autosp_set_error("bad shape b=%d s=%d d=%d elem_bytes=%d", b, s_global, d, elem_bytes);
    return AUTOSP_ERR_VALIDATION;
  }
  if (s_global % world) {
    autosp_set_error("sequence %d not divisible by world size %d", s_global, world);
    return AUTOSP_ERR_VALIDATION;
  }
  if (!peer_base || !peer_flags) {
    autosp_set_error("peer_base / peer_flags must be non-null");
    return AUTOSP_ERR_VALIDATION;
  }
  A2AParams p{};
  p.n = n_tensors;
  p.dir = direction;
  p.b = b;
  p.s_glob = s_global;
  p.s_loc = s_global / world;
  p.d = d;
  p.eb = elem_bytes;
  p.P = world;
  p.rank = rank;
  p.epoch = epoch;
  p.timeout_ns = g_spin_timeout_ns;
  p.check = autosp_a2a_check(direction, tensors, n_tensors);
  for (int j = 0; j < world; ++j) {
    p.peer_base[j] = static_cast<char*>(peer_base[j]);
    p.peer_flags[j] = peer_flags[j];
    if (!p.peer_base[j] || !p.peer_flags[j]) {
      autosp_set_error("peer %d base/flags pointer is null", j);
      return AUTOSP_ERR_VALIDATION;
    }
  }
  // widest vector that divides every row / stride / pointer
  uint64_t align = 16;  // power of two dividing every row / stride / pointer
  auto fold = [&](uint64_t v) { while (align > 1 && (v % align)) align >>= 1; };
  fold((uint64_t)d * elem_bytes);
  for (int j = 0; j < world; ++j) fold((uint64_t)(uintptr_t)p.peer_base[j]);
  const int s_src = direction == AUTOSP_SEQ_TO_HEAD ? p.s_loc : s_global;
  p.total_items = 0;
  for (int i = 0; i < n_tensors; ++i) {
    const autosp_a2a_tensor& T = tensors[i];
    if (T.heads < 1 || !T.src) {
      autosp_set_error("tensor %d: heads must be positive and src non-null", i);
      return AUTOSP_ERR_VALIDATION;
    }
    if (direction == AUTOSP_SEQ_TO_HEAD && T.heads % world) {
      autosp_set_error("heads %d not divisible by world size %d", T.heads, world);
      return AUTOSP_ERR_VALIDATION;
    }
    A2ATensorDev& D = p.t[i];
    D.src = static_cast<const char*>(T.src);
    D.ss_b = T.src_stride_b; D.ss_s = T.src_stride_s; D.ss_h = T.src_stride_h;
    D.dst_off = T.dst_offset;
    D.ds_b = T.dst_stride_b; D.ds_s = T.dst_stride_s; D.ds_h = T.dst_stride_h;
    D.heads = T.heads;
    D.rope = T.rope ? 1 : 0;
    D.tiles = (s_src + kTileTokens - 1) / kTileTokens;
    D.items = (int64_t)b * T.heads * D.tiles;
    p.total_items += D.items;
    fold((uint64_t)(uintptr_t)T.src);
    fold((uint64_t)T.dst_offset);
    for (int64_t st : {T.src_stride_b, T.src_stride_s, T.src_stride_h, T.dst_stride_b,
                       T.dst_stride_s, T.dst_stride_h})
      fold((uint64_t)(st < 0 ? -st : st) * elem_bytes);
  }
  const uint64_t row = (uint64_t)d * elem_bytes;
  if (row / align > 32) {
    autosp_set_error("row of %llu bytes needs >32 lanes at %llu-byte granularity (unsupported)",
                     (unsigned long long)row, (unsigned long long)align);
    return AUTOSP_ERR_UNSUPPORTED;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t warps_needed = p.total_items;
  int64_t blocks = (warps_needed + (kA2AThreads / 32) - 1) / (kA2AThreads / 32);
  const int64_t max_blocks = (int64_t)sms * AUTOSP_A2A_BPS;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (world > 1) a2a_handshake_kernel<<<1, 32, 0, st>>>(p);
  const bool fast = align == 16 && (row == 64 || row == 128 || row == 256) &&
                    p.total_items < (int64_t)INT32_MAX;
  p.pos = pos;
  p.log2_theta = pos ? log2f(theta) : 0.f;
  if (pos && !fast) {
    autosp_set_error("a2a with RoPE needs 16-byte aligned rows of 64/128/256 bytes");
    return AUTOSP_ERR_UNSUPPORTED;
  }
  if (fast) {
    switch (row) {
      case 64: a2a_push_fast<64><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
      case 128: a2a_push_fast<128><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
      default: a2a_push_fast<256><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
    }
  } else switch (align) {
    case 16: a2a_push_kernel<uint4><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
    case 8: a2a_push_kernel<uint2><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
    case 4: a2a_push_kernel<uint32_t><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
    default: a2a_push_kernel<uint16_t><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    autosp_set_error("a2a launch failed: %s", cudaGetErrorString(e));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}

extern "C" int autosp_a2a_grad_out(const autosp_a2a_tensor* t2, int b, int s_global, int d,
                                   int world, int rank, void* const* peer_base,
                                   uint32_t* const* peer_flags, uint32_t epoch, void* stream) {
  using namespace autosp;
  if (!t2 || !t2[0].src || !t2[1].src || (d != 32 && d != 64 && d != 128) || b < 1 ||
      world < 1 || world > AUTOSP_MAX_WORLD || rank < 0 || rank >= world || s_global % world ||
      t2[0].heads < 1 || t2[0].heads % world || t2[1].heads != t2[0].heads || !peer_base ||
      !peer_flags) {
    autosp_set_error("a2a_grad_out: bad arguments (d=%d world=%d rank=%d)", d, world, rank);
    return AUTOSP_ERR_VALIDATION;
  }
  A2AParams p{};
  p.n = 2;
  p.dir = AUTOSP_SEQ_TO_HEAD;
  p.b = b;
  p.s_glob = s_global;
  p.s_loc = s_global / world;
  p.d = d;
  p.eb = 2;
  p.P = world;
  p.rank = rank;
  p.epoch = epoch;
  p.timeout_ns = g_spin_timeout_ns;
  p.check = autosp_a2a_check(AUTOSP_SEQ_TO_HEAD, t2, 2);
  uint64_t align = 0;
  for (int i = 0; i < 2; ++i) {
    const autosp_a2a_tensor& T = t2[i];
    A2ATensorDev& D = p.t[i];
    D.src = static_cast<const char*>(T.src);
    D.ss_b = T.src_stride_b; D.ss_s = T.src_stride_s; D.ss_h = T.src_stride_h;
    D.dst_off = T.dst_offset;
    D.ds_b = T.dst_stride_b; D.ds_s = T.dst_stride_s; D.ds_h = T.dst_stride_h;
    D.heads = T.heads;
    D.tiles = (p.s_loc + kTileTokens - 1) / kTileTokens;
    D.items = (int64_t)b * T.heads * D.tiles;
    align |= (uint64_t)(uintptr_t)T.src | (uint64_t)(T.src_stride_b | T.src_stride_s |
                                                      T.src_stride_h) * 2;
  }
  align |= (uint64_t)t2[0].dst_offset | (uint64_t)(t2[0].dst_stride_b | t2[0].dst_stride_s |
                                                   t2[0].dst_stride_h) * 2;
  align |= (uint64_t)(t2[1].dst_offset & 3);
  if (align & 15) {
    autosp_set_error("a2a_grad_out: sources / dO destination must be 16-byte aligned rows "
                     "(delta destination 4-byte aligned)");
    return AUTOSP_ERR_VALIDATION;
  }
  for (int j = 0; j < world; ++j) {
    if (!peer_base[j] || !peer_flags[j] || (reinterpret_cast<uintptr_t>(peer_base[j]) & 15)) {
      autosp_set_error("a2a_grad_out: peer %d base/flags null or misaligned", j);
      return AUTOSP_ERR_VALIDATION;
    }
    p.peer_base[j] = static_cast<char*>(peer_base[j]);
    p.peer_flags[j] = peer_flags[j];
  }
  p.total_items = p.t[0].items;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int64_t blocks = (p.total_items + (kA2AThreads / 32) - 1) / (kA2AThreads / 32);
  if (blocks > (int64_t)sms * 4) blocks = (int64_t)sms * 4;
  if (blocks < 1) blocks = 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (world > 1) a2a_handshake_kernel<<<1, 32, 0, st>>>(p);
  switch (d) {
    case 32: a2a_grad_out_kernel<64><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
    case 64: a2a_grad_out_kernel<128><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
    default: a2a_grad_out_kernel<256><<<(int)blocks, kA2AThreads, 0, st>>>(p); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    autosp_set_error("a2a_grad_out launch failed: %s", cudaGetErrorString(e));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}

extern "C" uint32_t autosp_a2a_check(int direction, const autosp_a2a_tensor* tensors,
                                     int n_tensors) {
  autosp::CheckHash h;
  h.add(direction);
  h.add(n_tensors);
  for (int i = 0; tensors && i < n_tensors; ++i) {
    const autosp_a2a_tensor& T = tensors[i];
    h.add(T.dst_offset);
    h.add(T.dst_stride_b);
    h.add(T.dst_stride_s);
    h.add(T.dst_stride_h);
    h.add(T.heads);
  }
  return h.h;
}

extern "C" uint32_t autosp_push_check(const autosp_push_spec* push, int heads) {
  if (!push) return 0u;
  autosp_a2a_tensor t{};
  t.dst_offset = push->dst_offset;
  t.dst_stride_b = push->dst_stride_b;
  t.dst_stride_s = push->dst_stride_s;
  t.dst_stride_h = push->dst_stride_h;
  t.heads = heads;
  return autosp_a2a_check(AUTOSP_HEAD_TO_SEQ, &t, 1);
}

extern "C" int autosp_a2a_wait(uint32_t* local_flags, int world, int rank, uint32_t epoch,
                               uint32_t check, void* stream) {
  if (!local_flags || world < 1 || world > AUTOSP_MAX_WORLD || rank < 0 || rank >= world) {
    autosp_set_error("bad a2a_wait arguments (world %d rank %d)", world, rank);
    return AUTOSP_ERR_VALIDATION;
  }
  if (world == 1) return AUTOSP_OK;
  autosp::a2a_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      local_flags, world, rank, epoch, check, g_spin_timeout_ns);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    autosp_set_error("a2a_wait launch failed: %s", cudaGetErrorString(e));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}

extern "C" int autosp_a2a_mark_ready(uint32_t* const* flags, int world, uint32_t epoch,
                                     void* stream) {
  if (!flags || world < 1 || world > AUTOSP_MAX_WORLD) {
    autosp_set_error("bad mark_ready arguments");
    return AUTOSP_ERR_VALIDATION;
  }
  autosp::MarkParams m{};
  for (int j = 0; j < world; ++j) m.flags[j] = flags[j];
  m.P = world;
  m.epoch = epoch;
  autosp::a2a_mark_ready_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(m);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    autosp_set_error("mark_ready launch failed: %s", cudaGetErrorString(e));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}

// Ready handshake before a fused compute+push kernel (same protocol as the a2a calls).
int autosp_internal_handshake(uint32_t* const* flags, int world, int rank, uint32_t epoch,
                              cudaStream_t stream) {
  autosp::ShakeParams s{};
  for (int j = 0; j < world; ++j) s.flags[j] = flags[j];
  s.P = world;
  s.rank = rank;
  s.epoch = epoch;
  s.timeout_ns = g_spin_timeout_ns;
  autosp::handshake_kernel<<<1, 32, 0, stream>>>(s);
  return cudaGetLastError() == cudaSuccess ? AUTOSP_OK : AUTOSP_ERR_CUDA;
}

int autosp_preload_a2a() {
  cudaFuncAttributes h;
  cudaFuncGetAttributes(&h, autosp::handshake_kernel);
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, autosp::a2a_push_fast<64>);
  cudaFuncGetAttributes(&a, autosp::a2a_push_fast<128>);
  cudaFuncGetAttributes(&a, autosp::a2a_push_fast<256>);
  cudaFuncGetAttributes(&a, autosp::a2a_push_kernel<uint4>);
  cudaFuncGetAttributes(&a, autosp::a2a_push_kernel<uint2>);
  cudaFuncGetAttributes(&a, autosp::a2a_push_kernel<uint32_t>);
  cudaFuncGetAttributes(&a, autosp::a2a_push_kernel<uint16_t>);
  cudaFuncGetAttributes(&a, autosp::a2a_handshake_kernel);
  cudaFuncGetAttributes(&a, autosp::a2a_wait_kernel);
  cudaFuncGetAttributes(&a, autosp::a2a_mark_ready_kernel);
  cudaFuncGetAttributes(&a, autosp::a2a_grad_out_kernel<64>);
  cudaFuncGetAttributes(&a, autosp::a2a_grad_out_kernel<128>);
  cudaFuncGetAttributes(&a, autosp::a2a_grad_out_kernel<256>);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
