/*
 * autosp.h — C ABI of libautosp.so, the B200 (sm_100a) hot path of AutoSP's
 * Ulysses sequence parallelism.
 *
 * Plain pointers, sizes and an opaque `void* stream` (a cudaStream_t); no torch
 * types.  Every call is stream-ordered on `stream`, never allocates, never
 * synchronises the host, and returns an autosp_status.  The text of the last
 * error on the calling thread is available from autosp_last_error().
 *
 * Each entry point replaces one reference interface (paths relative to
 * /root/reference/pkg/src/seqcomp):
 *
 *   autosp_a2a            all_to_all_shards          executor.py:203-230
 *                         DeviceGroup.submit/take     executor.py:244-275
 *                         (the AllToAll node inserted by transform_sp, sp_pass.py:172-195,
 *                          and its gradient, autodiff.py:252-262)
 *   autosp_a2a_wait       DeviceGroup.ready           executor.py:267-268
 *   autosp_symm_*         DeviceGroup(P) rendezvous   executor.py:233-242
 *   autosp_attn_fwd       _eval_attention_core        executor.py:132-142
 *                         (lowered recipe lowering.py:82-122)
 *   autosp_attn_bwd       attention backward recipes  autodiff.py:156-162,190-195,213-214,
 *                                                     executor.py:89-91
 *   status codes          errors.py:4-29 (ValidationError/CollectiveError -> 2)
 */
#ifndef AUTOSP_H_
#define AUTOSP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AUTOSP_ABI_VERSION 3

#if defined(__GNUC__)
#define AUTOSP_API __attribute__((visibility("default")))
#else
#define AUTOSP_API
#endif

typedef enum autosp_status {
  AUTOSP_OK = 0,
  AUTOSP_ERR_INTERNAL = 1,   /* SeqcompError (errors.py:4-5)                       */
  AUTOSP_ERR_VALIDATION = 2, /* ValidationError / CollectiveError (errors.py:8-29)  */
  AUTOSP_ERR_UNSUPPORTED = 3,/* shape outside what the sm_100a kernels implement     */
  AUTOSP_ERR_CUDA = 5        /* CUDA runtime / driver failure                        */
} autosp_status;

typedef enum autosp_direction {
  AUTOSP_SEQ_TO_HEAD = 0, /* "seq_to_head" (sp_pass.py:175-180) */
  AUTOSP_HEAD_TO_SEQ = 1  /* "head_to_seq" (sp_pass.py:187-192) */
} autosp_direction;

AUTOSP_API int autosp_abi_version(void);
AUTOSP_API const char* autosp_last_error(void);
/* Load every kernel of the library into the current context now (instead of lazily at
 * first launch: a lazy module load can implicitly synchronise the context, which must
 * not happen while a peer's all-to-all is spinning on this GPU).                      */
AUTOSP_API int autosp_preload_kernels(void);
/* number of SMs / compute capability of the current device, -1 if no device */
AUTOSP_API int autosp_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------------ symmetric memory
 * One allocation per rank, identical size on every rank, mapped into every peer of the
 * SP group once at dist.init (CUDA IPC over NVLink/NVSwitch).  The handle is an opaque
 * 64-byte blob exchanged by the host (torch.distributed all_gather_object).           */
#define AUTOSP_IPC_HANDLE_BYTES 64
AUTOSP_API int autosp_symm_alloc(size_t bytes, void** dev_ptr, void* ipc_handle_out);
AUTOSP_API int autosp_symm_open(const void* ipc_handle, void** dev_ptr);
AUTOSP_API int autosp_symm_close(void* peer_ptr);
AUTOSP_API int autosp_symm_free(void* dev_ptr);
AUTOSP_API int autosp_memset_async(void* dev_ptr, int value, size_t bytes, void* stream);
/* A DLPack (v0.8 DLManagedTensor, capsule name "dltensor") 1-D uint8 view of `nbytes`
 * of memory owned by this library (receive-region slots), allocated in C with a C deleter
 * so the framework can drop the view at any time -- including interpreter shutdown --
 * without calling back into the host language.  device_type: 2 = CUDA, 1 = CPU. */
AUTOSP_API void* autosp_dlpack_wrap(void* ptr, int64_t nbytes, int device_type, int device_id);

/* ------------------------------------------------------------------ all-to-all reshard
 * One logical [b, s, h, d] tensor (head_dim d contiguous).  Strides are in ELEMENTS.
 *   seq_to_head: the source is this rank's sequence shard [b, s/P, h, d]; rank j receives
 *                heads [j*h/P, (j+1)*h/P) of every token, written at sequence offset
 *                rank*s/P of its destination [b, s, h/P, d].
 *   head_to_seq: the source is this rank's head block [b, s, h, d] (h = local heads);
 *                rank j receives tokens [j*s/P, (j+1)*s/P) written at head offset rank*h
 *                of its destination [b, s/P, h*P, d].
 * `dst_offset` is the byte offset of the destination tensor inside every rank's symmetric
 * receive region (identical on all ranks); dst strides describe that destination, so
 * the QKV-projection and O-projection layout transposes fold into the copy.          */
typedef struct autosp_a2a_tensor {
  const void* src;
  int64_t src_stride_b, src_stride_s, src_stride_h;
  int64_t dst_offset;
  int64_t dst_stride_b, dst_stride_s, dst_stride_h;
  int32_t heads; /* h of the SOURCE logical tensor */
  int32_t rope;  /* autosp_a2a_rope only: 1 = rotate (RoPE) the rows while moving them */
} autosp_a2a_tensor;

#define AUTOSP_A2A_MAX_TENSORS 4
#define AUTOSP_MAX_WORLD 8
#define AUTOSP_FLAG_WORDS 64 /* uint32 words of one rank's flag block */

/* Push this rank's slabs of up to 4 tensors straight into every peer's receive region
 * (16-byte vector stores over NVLink; the local slab is a local copy), then publish
 * `epoch` in every peer's flag block.  peer_base[j] / peer_flags[j] are rank j's
 * receive region / flag block as mapped in THIS process (peer_flags[rank] is local).
 * Before writing into rank j the kernel waits until rank j has itself reached `epoch`
 * (its previous readers of the region are stream-ordered before that point).
 * epoch must increase by one per call, identically on every rank.                   */
AUTOSP_API int autosp_a2a(int direction, const autosp_a2a_tensor* tensors, int n_tensors, int b,
               int s_global, int d, int elem_bytes, int world, int rank,
               void* const* peer_base, uint32_t* const* peer_flags, uint32_t epoch,
               void* stream);
/* autosp_a2a with RoPE folded into the reshard (seq_to_head, bf16, d in {32,64,128}):
 * tensors with rope = 1 are rotated (rotate-half, pos[t] of the source token t, theta)
 * on the way, so the projection output is read ONCE and arrives rotated and head-major
 * at its owner -- no separate RoPE / split / transpose kernel.                        */
AUTOSP_API int autosp_a2a_rope(int direction, const autosp_a2a_tensor* tensors, int n_tensors,
               int b, int s_global, int d, int elem_bytes, int world, int rank,
               void* const* peer_base, uint32_t* const* peer_flags, uint32_t epoch,
               const float* pos, float theta, void* stream);
/* The backward's seq->head reshard of the attention-output gradient fused with
 * delta = rowsum(dO * O) (softmax_dx's correction term, executor.py:89-91), formed on the
 * token owner: t2[0] = dO (token-major source, head-major [b, h/P, S, d] destination as in
 * autosp_a2a), t2[1] = O (token-major source, same logical shape) whose DESTINATION is the
 * fp32 delta [b, h/P, S] (dst strides in fp32 elements, dst_stride_s = 1).  bf16, d in
 * {32, 64, 128}.  One handshake + one push launch; the receiver waits with autosp_a2a_wait
 * (check = autosp_a2a_check(AUTOSP_SEQ_TO_HEAD, t2, 2)).                              */
AUTOSP_API int autosp_a2a_grad_out(const autosp_a2a_tensor* t2, int b, int s_global, int d,
               int world, int rank, void* const* peer_base, uint32_t* const* peer_flags,
               uint32_t epoch, void* stream);
/* Stream-ordered wait until every peer has published `epoch` into this rank's flag
 * block (the receive region then holds the complete a2a output).  `check` is the check
 * word of the call as THIS rank sees it (autosp_a2a_check of its descriptors, or
 * autosp_push_check for autosp_attn_fwd_push): every sender publishes the check word of
 * its own descriptors (all destination offsets, strides and head counts of the call) and
 * the wait traps on any disagreement (symmetric-allocation invariant).              */
AUTOSP_API int autosp_a2a_wait(uint32_t* local_flags, int world, int rank, uint32_t epoch,
                               uint32_t check, void* stream);
AUTOSP_API uint32_t autosp_a2a_check(int direction, const autosp_a2a_tensor* tensors,
                                     int n_tensors);
/* Every flag spin of the reshard protocol (waiting for a peer to reach an epoch or to
 * finish writing) traps after this many seconds instead of hanging the GPU; default 300.
 * Host-side setting, applies to launches issued after the call.                       */
AUTOSP_API int autosp_set_spin_timeout(double seconds);
/* Single-process loopback used by tests / benchmarks on one GPU: marks `epoch` as reached
 * for all `world` virtual ranks whose flag blocks are given.                           */
AUTOSP_API int autosp_a2a_mark_ready(uint32_t* const* flags, int world, uint32_t epoch, void* stream);

/* ------------------------------------------------------------------ causal attention
 * q [b, hq, s, d], k/v [b, hkv, s, d] as strided views (d contiguous, element strides in
 * (b, h, s) order; 16-byte aligned), bf16.  GQA: q head i reads kv head i / (hq/hkv).
 * o is written in the same convention; lse [b, hq, s] fp32 (natural log of the row sum
 * of exp(scale * q.k) over unmasked keys).  d in {32, 64, 128}.                      */
typedef struct autosp_attn_tensor {
  const void* ptr;
  int64_t stride_b, stride_h, stride_s;
} autosp_attn_tensor;

AUTOSP_API int autosp_attn_fwd(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                    autosp_attn_tensor o, float* lse, int b, int hq, int hkv, int s, int d,
                    float scale, int causal, void* stream);

/* Fused K3 + K2: the attention forward ALSO pushes every output row to the rank that owns
 * its token (the head->seq all-to-all of O, reference executor.py:222-229) from the
 * epilogue, over the same symmetric regions / epoch protocol as autosp_a2a, so the
 * transfer overlaps the attention math tile by tile and no separate reshard kernel
 * reads O back.  q/k/v/o/lse as in autosp_attn_fwd over the FULL sequence s on this
 * rank's hq heads; row (b, h, t) lands in rank t / (s / world) at byte offset
 * dst_offset + 2 * (b * dst_stride_b + (t mod s/world) * dst_stride_s
 *                   + (rank * hq + h) * dst_stride_h)
 * of its receive region.  Publishes arrive flags like autosp_a2a; the caller then runs
 * autosp_a2a_wait.  Replaces the autosp_attn_fwd + autosp_a2a(head_to_seq) pair.
 * o.ptr may be NULL: only the pushed (token-major) copy is written. */
typedef struct autosp_push_spec {
  int world, rank;
  int64_t dst_offset;                          /* bytes, identical on every rank */
  int64_t dst_stride_b, dst_stride_s, dst_stride_h;  /* elements */
  void* const* peer_base;                      /* [world] receive regions */
  uint32_t* const* peer_flags;                 /* [world] flag blocks */
  uint32_t epoch;
} autosp_push_spec;

/* check word of an autosp_attn_fwd_push call on `heads` local heads (see autosp_a2a_wait) */
AUTOSP_API uint32_t autosp_push_check(const autosp_push_spec* push, int heads);
AUTOSP_API int autosp_attn_fwd_push(autosp_attn_tensor q, autosp_attn_tensor k,
                    autosp_attn_tensor v, autosp_attn_tensor o, float* lse, int b, int hq,
                    int hkv, int s, int d, float scale, int causal,
                    const autosp_push_spec* push, void* stream);

/* fp32 workspace the backward needs: dq accumulator [b, hq, s, d] + delta [b, hq, s]
 * + -lse*log2(e) [b, hq, s] (+ dK/dV partials [2, b, hkv, s, d] when the launch splits
 * each kv head's q-head group over two CTAs to fill the GPU: small grids, GQA) */
AUTOSP_API size_t autosp_attn_bwd_workspace_bytes(int b, int hq, int hkv, int s, int d);
AUTOSP_API int autosp_attn_bwd(autosp_attn_tensor q, autosp_attn_tensor k, autosp_attn_tensor v,
                    autosp_attn_tensor o, autosp_attn_tensor d_o, const float* lse,
                    autosp_attn_tensor dq, autosp_attn_tensor dk, autosp_attn_tensor dv,
                    void* workspace, int b, int hq, int hkv, int s, int d, float scale,
                    int causal, void* stream);

/* autosp_attn_bwd with delta[b, hq, s] = rowsum(dO * O) (fp32, contiguous) supplied by the
 * caller instead of O: the Ulysses backward forms delta on the token owner from the
 * token-major output it keeps anyway and reshards it with dO, so the head-major O need
 * not be kept for the backward. */
AUTOSP_API int autosp_attn_bwd_delta(autosp_attn_tensor q, autosp_attn_tensor k,
                    autosp_attn_tensor v, const float* delta, autosp_attn_tensor d_o,
                    const float* lse, autosp_attn_tensor dq, autosp_attn_tensor dk,
                    autosp_attn_tensor dv, void* workspace, int b, int hq, int hkv, int s, int d,
                    float scale, int causal, void* stream);

/* autosp_attn_bwd_delta fused with the head->seq all-to-all of the gradients (the
 * backward of the RoPE-fused seq->head reshard, autodiff.py:252-262): nothing is written
 * locally; every dQ / dK / dV row goes straight into the token owner's receive region as
 * the PACKED QKV-projection gradient [b, s/P, hq*P + 2*hkv*P, d] (push->dst_* strides;
 * dq at global head rank*hq + h, dk at hq*P + rank*hkv + h, dv at hq*P + hkv*P + rank*hkv
 * + h; hq/hkv are this rank's local head counts).  The ready handshake runs first; the
 * arrival is published when the last dQ row is out.  Check word: autosp_push_check(push,
 * hq + 2*hkv).  The receiver waits with autosp_a2a_wait. */
AUTOSP_API int autosp_attn_bwd_push(autosp_attn_tensor q, autosp_attn_tensor k,
                    autosp_attn_tensor v, const float* delta, autosp_attn_tensor d_o,
                    const float* lse, void* workspace, int b, int hq, int hkv, int s, int d,
                    float scale, int causal, const autosp_push_spec* push, void* stream);

/* K0: the packed QKV projection Y = X W^T (X [M, K] bf16 with row stride ldx -- M = b * s_loc
 * tokens of this rank; W [N, K] with N = (hq + 2hkv) * d, the nn.Linear weight; fp32
 * accumulation in TMEM; tcgen05 + TMA, persistent) with the seq->head all-to-all folded
 * into its epilogue (replaces the projection Linear + AllToAll of transformer.py:66-72 /
 * executor.py:203-230 in the reference's lowered graph):
 *   dst3 != NULL: every (token, head) row is rounded to bf16, RoPE-rotated when it is a q
 *     or k head and rope != 0 (pos[t] of this rank's token t, theta; bit-identical to K1's
 *     rotation), and stored into the owning rank's receive region at dst3[i].dst_offset as
 *     the contiguous head-major [b, h/P, s_loc * world, d] operand (i = q, k, v; heads =
 *     hq / hkv / hkv GLOBAL head counts).  Ready handshake first; arrival published at the
 *     end; the receiver waits with autosp_a2a_wait(check = autosp_a2a_check(SEQ_TO_HEAD,
 *     dst3, 3)).
 *   dst3 == NULL: a plain GEMM into the local row-major Y (ldy >= N); rope must be 0.
 * Needs M % 128 == 0, s_loc % 128 == 0, N % 256 == 0, K % 64 == 0 (else status 3). */
AUTOSP_API int autosp_qkv_gemm(const void* x, int64_t ldx, const void* w, int64_t ldw, int M,
                    int K, int hq, int hkv, int d, int s_loc, const float* pos, float theta,
                    int rope, void* y, int64_t ldy, const autosp_a2a_tensor* dst3, int world,
                    int rank, void* const* peer_base, uint32_t* const* peer_flags,
                    uint32_t epoch, void* stream);

/* ------------------------------------------------------------------ fused elementwise
 * HBM-bound bf16 kernels for the layer around the Ulysses path (fp32 math):
 *   swiglu: out[r, :] = silu(gu[r, :F]) * gu[r, F:2F]        (reference silu executor.py:33-34,
 *           silu_dx :85-88);  bwd writes dgu = [dg | du]
 *   rope:   rotate-half RoPE of x [b, s, h, d] (strided) with angles pos[t] * theta^(-2i/d);
 *           inverse = 1 rotates by the negative angle (the backward)
 *   ce:     per-row log-sum-exp / cross entropy over bf16 logits [rows, vocab] (leading dim
 *           ld); ce_bwd overwrites the logits with g * (softmax - onehot(label)).  Rows whose
 *           label lies outside [0, vocab) (the -100 padding convention) are ignored: loss 0
 *           and an all-zero gradient row.                                                */
AUTOSP_API int autosp_swiglu_fwd(const void* gu, void* out, int64_t rows, int ffn, int64_t ld_gu,
                                 int64_t ld_out, void* stream);
AUTOSP_API int autosp_swiglu_bwd(const void* gu, const void* dout, void* dgu, int64_t rows,
                                 int ffn, int64_t ld_gu, int64_t ld_dout, int64_t ld_dgu,
                                 void* stream);
AUTOSP_API int autosp_rope(const void* x, void* y, int b, int s, int h, int d, int64_t xsb,
                           int64_t xss, int64_t xsh, int64_t ysb, int64_t yss, int64_t ysh,
                           const float* pos, float theta, int inverse, void* stream);
/* Segmented RoPE (rotate-half, positions pos[s], theta; inverse = rotate by -angle):
 * each segment maps a [b, s, heads, d] strided view src to dst, rotating when `rotate`
 * and copying otherwise.  Forward: the packed QKV projection output -> q, k (rotated), v;
 * backward: dq, dk (inverse rotation), dv -> the packed QKV gradient.  One launch. */
typedef struct autosp_rope_segment {
  const void* src;
  void* dst;
  int64_t src_stride_b, src_stride_s, src_stride_h;  /* elements */
  int64_t dst_stride_b, dst_stride_s, dst_stride_h;
  int heads, rotate;
} autosp_rope_segment;
AUTOSP_API int autosp_rope_segments(const autosp_rope_segment* segs, int nseg, int b, int s,
                                    int d, const float* pos, float theta, int inverse,
                                    void* stream);
/* RMSNorm (reference executor.py:43-45, eps inside the sqrt): y = x * rstd * w over rows
 * of d (bf16, leading dims in elements), rstd [rows] fp32.  Backward: dx and dw (bf16 [d])
 * in one pass over (dy, x) plus a column sum of per-CTA partials (workspace). */
AUTOSP_API int autosp_rms_norm_fwd(const void* x, const void* w, void* y, float* rstd,
                                   int64_t rows, int d, int64_t ld_x, int64_t ld_y, float eps,
                                   void* stream);
AUTOSP_API size_t autosp_rms_norm_bwd_workspace_bytes(int d);
AUTOSP_API int autosp_rms_norm_bwd(const void* dy, const void* x, const void* w,
                                   const float* rstd, void* dx, void* dw, void* workspace,
                                   int64_t rows, int d, int64_t ld_dy, int64_t ld_x,
                                   int64_t ld_dx, void* stream);
AUTOSP_API int autosp_ce_fwd(const void* logits, const int64_t* labels, float* lse, float* loss,
                             int64_t rows, int64_t vocab, int64_t ld, void* stream);
AUTOSP_API int autosp_ce_bwd(void* logits, const int64_t* labels, const float* lse, float g,
                             int64_t rows, int64_t vocab, int64_t ld, void* stream);

/* Multi-tensor AdamW for bf16 parameters with bf16 moments (the optimizer step of the
 * training loop the bench times; not part of the reference, whose workload has no
 * optimizer).  Same update order as torch.optim.AdamW: p *= 1 - lr*wd; m = lerp(m, g, 1-b1);
 * v = b2 v + (1-b2) g^2; p -= lr/(1-b1^t) * m / (sqrt(v)/sqrt(1-b2^t) + eps), fp32 math.
 * `tensors` is a host array; up to 64 tensors per kernel launch. */
typedef struct {
  void* p;
  const void* g;
  void* m;
  void* v;
  int64_t n;
} autosp_adamw_tensor;
AUTOSP_API int autosp_adamw_bf16(const autosp_adamw_tensor* tensors, int count, float lr,
                                 float beta1, float beta2, float eps, float weight_decay,
                                 int step, void* stream);

/* debug only: per-step timeline of the backward's first CTA into dev_buf (16 x 64 int64) */
AUTOSP_API int autosp_debug_set_bwd_trace(long long* dev_buf);
AUTOSP_API int autosp_debug_set_fwd_trace(long long* dev_buf);

#ifdef __cplusplus
}
#endif
#endif /* AUTOSP_H_ */
