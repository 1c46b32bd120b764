/*
 * mace_b200.h — C-ABI of libmace_b200.so, the sm_100a execution layer for MACE's hybrid iteration.
 *
 * The reference (macesim, a discrete-event simulator) has no native layer: every entry point below
 * replaces a cost-model *stand-in* inside the reference's hot path, named per function:
 *   Engine._execute              /root/reference/pkg/src/macesim/engine.py:573-676
 *   Engine._exec_prefill         engine.py:444-480   (prefill rows: latency = 0.5 ms/token stand-in)
 *   Engine._exec_decode          engine.py:482-532   (decode rows: 20 ms/step stand-in, KV growth + prune)
 *   Engine._exec_ft / ft_step    engine.py:534-536, alignment.py:168-172 (mu += ft_gain stand-in)
 *   dpo_loss                     alignment.py:39-47  (the scalar stage shared with the fused DPO kernel)
 *   PrefixTrie.lru_offload       cache.py:217-238    (evict decision -> page free)
 *   prune trim                   engine.py:506-529   (kept[h] trim -> page-table compaction)
 * The Python side calls these through ctypes from GpuEngine._execute (the override point the reference
 * exposes, engine.py:573); see INTEGRATION.md for the binding.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes; `stream` is a cudaStream_t passed as void*.
 *  - The caller owns ALL device memory (weights, KV pools, activations, workspaces); kernels never
 *    allocate.
 *  - Every call is stream-ordered and asynchronous; returns 0 (MACE_OK) or a negative mace_status,
 *    with a message available from mace_last_error(ctx). No exceptions cross the ABI.
 *  - No process-global mutable state: one mace_ctx per Engine / thread (threaded sweeps are safe).
 *  - There is no CPU fallback: without a B200 (sm_100) device, mace_ctx_create fails.
 */
#ifndef MACE_B200_H
#define MACE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mace_ctx mace_ctx;
typedef struct mace_model mace_model;  /* native tick executor (section 5) */

enum mace_status {
  MACE_OK = 0,
  MACE_ERR_ARG = -1,
  MACE_ERR_CUDA = -2,
  MACE_ERR_LAUNCH = -3,
  MACE_ERR_NOMEM = -4,
  MACE_ERR_UNSUPPORTED = -5,
};

/* ---------------------------------------------------------------- context */
int mace_version(void);
int mace_ctx_create(int device, mace_ctx** out);
int mace_ctx_destroy(mace_ctx* ctx);
const char* mace_last_error(mace_ctx* ctx);
/* number of kernels this ctx has launched (evidence for the bench's gpu_launches) */
long long mace_launch_count(mace_ctx* ctx);
/* host issue profile, process-wide, enabled by MACE_HOST_PROF=1 at load: out[4] = seconds in kernel launches,
 * launches, seconds in tensor-map encodes, encodes, since the previous call (then reset); -1 when disabled */
int mace_debug_host_prof(double* out4);

/* ---------------------------------------------------------------- (2) bf16 tcgen05 GEMM
 * C[M,N] = alpha * A[M,K] . B[N,K]^T (+bias[N]).  A is stored K-major ([M, lda]) or, with
 * a_mn_major, MN-major ([K, lda], i.e. A^T row-major); same for B.  Epilogue modes: */
enum mace_epilogue {
  MACE_EPI_BF16 = 0,       /* out bf16 = result                                  */
  MACE_EPI_F32 = 1,        /* out fp32 = result                                  */
  MACE_EPI_F32_ADD = 2,    /* out fp32 += result (residual stream, grad accumulate) */
  MACE_EPI_F32_ATOMIC = 3, /* out fp32 += result via atomics (shared destination)   */
  MACE_EPI_BF16_GELU = 4,  /* out bf16 = gelu_tanh(result) (fused GPT-2 MLP activation) */
  MACE_EPI_BF16_SWIGLU = 5,/* out bf16 [M, N] = silu(A.Bg^T) * (A.Bu^T) with B = [gate rows 0..N-1; up rows
                              N..2N-1] (K-major, no bias): the fused Llama MLP activation */
  MACE_EPI_ARGMAX = 6,     /* greedy decode head: out = uint64 keys [M], ZEROED before the call; every row's key is
                              atomically max-reduced to (orderable fp32 bits of its largest result << 32) |
                              (0xffffffff - first column holding it), i.e. the argmax over N with the lowest index on
                              ties, without materialising the [M, N] logits (ldo, bias unused; no split-K).
                              mace_argmax_keys turns the keys into token ids and re-zeroes them. */
};
typedef struct MaceGemmArgs {
  const void* a; int lda; int a_mn_major;
  const void* b; int ldb; int b_mn_major;
  int M, N, K;
  void* out; int ldo; int mode;
  const void* bias;      /* bf16 [N] or NULL (added once) */
  float alpha;           /* 0 means 1 */
  int split_k;           /* 0 = heuristic */
  void* workspace;       /* fp32 scratch for split-K with bf16 output (may be NULL) */
  size_t workspace_bytes;
  int flags;             /* MACE_GEMM_B_STATIC: B is not written by the preceding kernel on the stream
                            (weights), so its first tiles are fetched before the PDL wait            */
} MaceGemmArgs;
#define MACE_GEMM_B_STATIC 1
int mace_gemm_bf16(mace_ctx* ctx, const MaceGemmArgs* args, void* stream);


/* ---------------------------------------------------------------- tick row tables
 * One hybrid tick = one ragged batch of rows: [prefill rows | decode rows | fine-tune rows].
 * Row order inside each group follows Engine._execute (engine.py:578-584): prefills in trie-DFS
 * order, decodes by id, fine-tunes by id. A "sequence" is a contiguous run of rows:
 *   kind 0 PREFILL : rows = uncached prompt suffix [n_pv - q_len, n_pv), KV in prompt pages
 *   kind 1 DECODE  : 1 row, KV = prompt[:n_pv] + per-head decode window [dec_first[h], dec_end)
 *   kind 2 FT      : rows = [prompt | response], dense causal KV read from the qkv rows          */
#define MACE_PAGE_TOKENS 16
typedef struct MaceSeq {
  int kind, q_start, q_len, slot; /* slot: KV-table slot of the request (paged kinds) */
  int n_pv;                       /* prompt tokens visible to this sequence            */
  int kv_len;                     /* FT / prefill: total causal KV length               */
  int hole0, hole_len;            /* FT: keys [hole0, hole0 + hole_len) are invisible to the rows at or after
                                     hole0 + hole_len (causal otherwise). A preference pair is ONE sequence
                                     [prompt | chosen | prompt[-1] | rejected]: hole0 = P - 1, hole_len = 1 +
                                     n_chosen, so the rejected branch attends to prompt[:-1], its own copy of
                                     the last prompt token and itself -- the prompt rows are computed once for
                                     both responses. 0, 0 for every other kind.                              */
} MaceSeq;

/* Device-resident KV page tables (persist across ticks).  Pools are head-major pages:
 *   pool[layer][page][MACE_PAGE_TOKENS][head_dim] bf16, one pool for K and one for V.
 * Prompt pages are allocated in groups of n_kv_heads (head page = group*Hkv + h) by the host page
 * manager (trie-owned, refcounted; PrefixTrie semantics cache.py:67-241).  Decode pages are per head,
 * popped from / pushed to a device free stack (mace_kv_decode_alloc / mace_kv_trim).            */
typedef struct MaceKvLayout {
  const int* ptab; int max_prompt_pages;   /* [slots][max_prompt_pages] prompt group ids */
  int* dtab; int max_dec_pages;            /* [slots][Hkv][max_dec_pages] decode ring    */
  int* dec_base;                           /* [slots][Hkv] decode slot held by dtab[..][0] row 0 */
  int* dec_first;                          /* [slots][Hkv] first retained decode slot    */
  int* dec_end;                            /* [slots] decode slots created               */
  int* free_stack; int* free_top; int stack_cap; /* device free list of decode head pages; free_top -> int[2]
                                                     = {stack top, status (bit 0: a pop found it empty)} */
  int n_kv_heads; int sink_page;           /* sink_page: reserved head page outside the stack that an
                                              exhausted pop points a row at (in-bounds, flagged in status) */
} MaceKvLayout;

/* ---------------------------------------------------------------- row kernels */
/* tokens[i] < 0 reads last_token[-tokens[i]-1] (the slot's previous greedy token, kept on device) */
int mace_embed(mace_ctx* ctx, const int* tokens, const int* pos, const int* last_token, const void* emb,
               const void* pos_emb, int T, int d, float* x, void* stream);
int mace_norm(mace_ctx* ctx, const float* x, int ldx, const int* rows, int n_rows, int d, const void* w,
              const void* b, int layernorm, float eps, void* out, int ldo, float* rstd_out, void* stream);
/* mace_rope_kv resolves each row's KV page from the row / sequence / page tables before its PDL wait: those
 * tables must not be written by either of the two kernels launched just before it on the stream (the tick
 * writes them before its first layer). */
int mace_rope_kv(mace_ctx* ctx, void* qkv, int T, int Hq, int Hkv, int hd, const int* row_pos, const int* row_seq,
                 const int* row_kvi, const MaceSeq* seqs, const float* cos_t, const float* sin_t, int apply_rope,
                 const MaceKvLayout* kv, void* k_pool, void* v_pool, void* stream);
int mace_act(mace_ctx* ctx, const void* u, int T, int F, int swiglu, void* out, void* stream);
int mace_argmax(mace_ctx* ctx, const float* logits, int n, int V, int ld, int* out, void* stream);
/* keys of a MACE_EPI_ARGMAX GEMM -> out[i] = argmax column of row i; keys[0..n) are reset to 0 (ready for the
 * next call). Same result as mace_argmax over the materialised fp32 logits (first index on ties). */
int mace_argmax_keys(mace_ctx* ctx, unsigned long long* keys, int n, int* out, void* stream);

/* ---------------------------------------------------------------- (1) ragged paged attention fwd
 * Prefill and fine-tune sequences run as tcgen05 tiles (128 query rows x one query head; S = QK^T
 * and O = PV on the tensor cores, K/V pages TMA-staged, online softmax in registers); decode
 * sequences run as bandwidth-bound warp items streaming K/V page pairs with cp.async.bulk.
 * Work lists are built per tick by the host:
 *   tc_items  int4 [n_tc]  = (seq, q_head, q_block, 0)
 *   dec_items int4 [n_dec] = (seq, kv_head, chunk << 16 | n_chunks, partial_base), ordered longest
 *             first; warps take items dynamically from the ticket counter dec_work (zero between
 *             launches: the warp drawing a launch's final ticket resets it). Multi-chunk
 *             partials go to
 *             dec_workspace[partial_base + chunk] ((2G + G*hd) fp32 each) and are merged in chunk
 *             order; dec_counters is a zero-initialised int [slots * Hkv] left zeroed.            */
typedef struct MaceAttnArgs {
  void* qkv; int T; int Hq; int Hkv; int hd; /* packed [T, (Hq+2Hkv)*hd] bf16 after RoPE */
  const MaceSeq* seqs;
  const int* tc_items; int n_tc;
  const int* dec_items; int n_dec;
  MaceKvLayout kv;
  const void* k_pool; const void* v_pool; long long pool_pages; /* this layer */
  void* out;          /* [T, Hq*hd] bf16 */
  float* lse;         /* [T, Hq] natural-log LSE (tc rows) or NULL */
  float* head_norm;   /* [T, Hq] ||o_{t,h}||_2 of decode rows or NULL */
  float scale;        /* softmax scale, 0 -> 1/sqrt(hd) */
  void* dec_workspace; size_t dec_workspace_bytes;
  int* dec_counters;
  unsigned long long* dec_work;  /* zero-initialised ticket counter, owned by the caller; each launch leaves it zero */
  int decode_impl;    /* 0 auto, 1 CUDA-core streaming kernel, 2 tcgen05 swap-AB kernel */
  int tc_pairs;       /* 1: tc_items are (seq, q_head, q_block PAIR p -> rows [256p, 256p + 256), kv tiles): the
                         two-query-tile kernel (head_dim 64 / 128); 0: (seq, q_head, q_block, kv tiles)  */
} MaceAttnArgs;
int mace_attn_fwd(mace_ctx* ctx, const MaceAttnArgs* args, void* stream);

/* ---------------------------------------------------------------- (3) fused DPO + masked AdamW
 * logits fp32 [R, ld] for the response-predicting rows of the tick's FT sequences; targets [R];
 * pair_rows [n_pairs][4] = (chosen_row0, n_chosen, rejected_row0, n_rejected); row_ps[R] = 2*pair+side.
 * ref_lp [n_pairs][2] (NULL: only the policy log-probs lp_out are produced, e.g. for the pi_ref pass).
 * Outputs: loss/margin [n_pairs] (loss = softplus(-beta m), alignment.py:39-47), coef [n_pairs][2]
 * and, if dlogits != NULL, dlogits bf16 [R, ldd] = d(mean loss)/d logits.                          */
int mace_dpo_fused(mace_ctx* ctx, const float* logits, int R, int V, int ld, const int* targets, const int* pair_rows,
                   int n_pairs, const int* row_ps, const float* ref_lp, float beta, float* row_lse, float* row_lp,
                   float* lp_out, float* loss, float* margin, float* coef, void* dlogits, int ldd, void* stream);
/* the scalar stage alone, fp64 (same device function the pair stage of mace_dpo_fused uses): per sample
 * margin = delta_plus - delta_minus, loss = dpo_loss(margin, beta) (alignment.py:39-47, same branches and
 * expression order), sig = sigma(-beta*margin). margin / sig may be NULL.                                  */
int mace_dpo_scalar(mace_ctx* ctx, const double* delta_plus, const double* delta_minus, const double* beta, int n,
                    double* loss, double* margin, double* sig, void* stream);
/* AdamW over arbitrary segments of the flat fp32 buffers (per-tenant LoRA adapters: one tenant's rows of every
 * stacked adapter): segment s covers master[seg_flat[s] .. + len_s) with len_s = seg_vstart[s+1] - seg_vstart[s]
 * (device int64 arrays; seg_vstart[0] = 0), bf16 copy seg_weights[s]. Same per-element arithmetic as
 * mace_adamw_masked2; float4 path when every offset / length is a multiple of 4 (vec4 != 0).                 */
int mace_adamw_segments(mace_ctx* ctx, float* master, float* m, float* v, const float* grad, int n_seg,
                        const long long* seg_vstart, const long long* seg_flat, void* const* seg_weights, long long n,
                        double lr, double beta1, double beta2, double eps, double weight_decay, int step, int vec4,
                        void* stream);
/* masked AdamW over the selected-parameter segments: flat fp32 master/m/v/grad [n]; segment s covers
 * [seg_offsets[s], seg_offsets[s+1]) and its bf16 working copy is seg_weights[s] (device array of
 * device pointers). torch.optim.AdamW update order; step is 1-based.                               */
int mace_adamw_masked(mace_ctx* ctx, float* master, float* m, float* v, const float* grad, long long n,
                      const long long* seg_offsets, void* const* seg_weights, int n_seg, float lr, float beta1,
                      float beta2, float eps, float weight_decay, int step, void* stream);
/* same update with double hyper-parameters (the fp32 scalars of the update are derived from them in double and
 * rounded once, as torch.optim.AdamW does from its Python floats); vec4 != 0 selects the float4 streaming kernel
 * when n and the fp32 buffers allow it -- the caller guarantees every seg_offsets[s] % 4 == 0 and every bf16 copy
 * 8-byte aligned. Bit-identical to vec4 = 0.                                                                 */
int mace_adamw_masked2(mace_ctx* ctx, float* master, float* m, float* v, const float* grad, long long n,
                       const long long* seg_offsets, void* const* seg_weights, int n_seg, double lr, double beta1,
                       double beta2, double eps, double weight_decay, int step, int vec4, void* stream);

/* ---------------------------------------------------------------- FT-row backward pieces */
int mace_norm_bwd(mace_ctx* ctx, const float* x, int ldx, const int* xrows, const float* dy, int lddy, int n, int d,
                  const void* w, int layernorm, float eps, float* dx, int lddx, const int* dxrows, float* dw, float* db,
                  float* workspace, size_t workspace_bytes, void* stream);
int mace_colsum_bf16(mace_ctx* ctx, const void* y, int n, int N, int ld, float* out, float* workspace,
                     size_t workspace_bytes, void* stream);
int mace_act_bwd(mace_ctx* ctx, const void* u, const void* da, int n, int F, int swiglu, void* du, void* stream);
int mace_rope_bwd(mace_ctx* ctx, float* dqkv, int n, int Hq, int Hkv, int hd, const int* pos, const float* cos_t,
                  const float* sin_t, void* stream);
int mace_f32_to_bf16(mace_ctx* ctx, const float* x, long long n, void* y, void* stream);
/* LoRA row mask: out[i, c] = bf16(scale * z[i, c]) if c / rank == tenant[i] else 0, for c < R (tenant NULL:
 * every column 0 -- the pi_ref pass). z fp32 [n, ldz], out bf16 [n, ldo]; R % 8 == 0.                       */
int mace_lora_mask(mace_ctx* ctx, const float* z, int ldz, const int* tenant, int n, int rank, int R, float scale,
                   void* out, int ldo, void* stream);
/* LoRA helpers: strided fp32 -> bf16 ([n, cols], cols % 8 == 0), and the scatter of adapter B^T rows [rows, out]
 * (bf16, row-major) into columns [col0, col0 + rows) of an augmented weight [out, ldd] ([W | B])               */
int mace_f32_to_bf16_2d(mace_ctx* ctx, const float* x, int ldx, int n, int cols, void* y, int ldy, void* stream);
int mace_lora_bt_scatter(mace_ctx* ctx, const void* bt, int rows, int out, void* dst, int ldd, int col0, void* stream);
/* widening copy; with mace_f32_to_bf16 it brackets the bf16 gradient all-reduce of lockstep replicas */
int mace_bf16_to_f32(mace_ctx* ctx, const void* x, long long n, float* y, void* stream);
/* attention backward of the dense causal FT sequences: items int4 [n_items] = (seq, kv_head, key_block, steps),
 * key blocks of 128 keys for head_dim 64 / 128 (tcgen05 kernel), 64 keys for head_dim 32; dqkv fp32 [n_rows, W]
 * zeroed by the caller (dQ accumulates across key blocks and GQA heads), dK / dV written.                     */
int mace_attn_bwd(mace_ctx* ctx, const void* qkv, const void* o, const void* dout, const float* lse, int n_rows, int Hq,
                  int Hkv, int hd, const MaceSeq* seqs, const int* items, int n_items, int row_offset, float* Dbuf,
                  float* dqkv, void* stream);
/* the same with a deterministic dQ: dq_order int32 [n_rows * Hq] zeroed once by the caller (left zeroed by every
 * call) orders the key blocks' dQ contributions of each (query block, query head) by ascending key block (an
 * acquire / release counter per block) instead of fp32 atomics, so dQ -- and the whole FT step -- is bitwise
 * reproducible. Items must be ordered by ascending key block within each (sequence, kv head) (LPT order is).   */
int mace_attn_bwd2(mace_ctx* ctx, const void* qkv, const void* o, const void* dout, const float* lse, int n_rows, int Hq,
                   int Hkv, int hd, const MaceSeq* seqs, const int* items, int n_items, int row_offset, float* Dbuf,
                   float* dqkv, int* dq_order, void* stream);

/* ---------------------------------------------------------------- (4) KV pages */
/* pages are popped per (slot, head) whose ring is full; the host mirrors the count and refuses a tick that
 * would exhaust the pool (KvCapacityError), so the sink page is a last line of defence only            */
int mace_kv_decode_alloc(mace_ctx* ctx, const MaceKvLayout* kv, const int* slots, int n, void* stream);
/* synchronous read of {stack top, status} (tests / post-mortem); status != 0 means a pop hit the sink   */
int mace_kv_status(mace_ctx* ctx, const MaceKvLayout* kv, int* out2);
int mace_kv_trim(mace_ctx* ctx, const MaceKvLayout* kv, const int* slots, const int* kept, int n, void* stream);
int mace_kv_release(mace_ctx* ctx, const MaceKvLayout* kv, const int* slots, int n, void* stream);
/* compaction (after mace_kv_trim): items int32 [n][2] = (slot, kv head) whose retained window [dec_first, dec_end)
 * (1 <= length <= max_w <= 64) fits in one page fewer when re-based -- the window's K/V rows move down to ring
 * offset 0 in every layer of both pools, dec_base = dec_first, and the emptied last ring page is pushed. The host
 * mirror (kvmanager.DecodePageMirror.compact) picks the items and counts the pages.                            */
int mace_kv_compact(mace_ctx* ctx, const MaceKvLayout* kv, const int* items, int n, int max_w, int n_layers, int hd,
                    long long pages_per_layer, void* k_pools, void* v_pools, void* stream);
int mace_kv_page_copy(mace_ctx* ctx, const int* copies, int n, int n_kv_heads, int hd, long long pages_per_layer,
                      int n_layers, void* k_pools, void* v_pools, void* stream);
int mace_kv_set_prompt_tables(mace_ctx* ctx, const MaceKvLayout* kv, const int* slots, const int* tables, int n,
                              int ncols, void* stream);
int mace_scatter_tokens(mace_ctx* ctx, const int* src, const int* slots, int n, int* last_token, void* stream);

/* ---------------------------------------------------------------- (5) native tick executor
 * One call issues a whole hybrid tick, i.e. the device work the reference charges for one bin in
 * Engine._execute (engine.py:573-676): page-table maintenance, embed, every decoder layer over the
 * ragged [prefill | decode | FT] batch, the decode head (final norm -> lm_head -> greedy token ->
 * last_token scatter) and, for FT rows, the pi_ref and policy sub-passes over the selected layers,
 * the fused DPO loss and the backward of the selected layers into the flat fp32 gradient.  The
 * optimizer step stays a separate call (mace_adamw_masked) so a gradient all-reduce can sit between.
 * All launches go to `stream` in order; nothing synchronizes.                                      */
typedef struct MaceLayerWeights {          /* bf16 device pointers; biases / norm bias NULL for llama */
  const void *attn_norm_w, *attn_norm_b, *qkv_w, *qkv_b, *o_w, *o_b;
  const void *mlp_norm_w, *mlp_norm_b, *up_w, *up_b, *down_w, *down_b;
} MaceLayerWeights;
typedef struct MaceLayerGrads {            /* fp32 views into the flat gradient (NULL: not trained) */
  float *attn_norm_w, *attn_norm_b, *qkv_w, *qkv_b, *o_w, *o_b;
  float *mlp_norm_w, *mlp_norm_b, *up_w, *up_b, *down_w, *down_b;
} MaceLayerGrads;
typedef struct MaceLoraLayer {             /* per-tenant LoRA adapters of one selected layer, tenants stacked:
                                              R = tenants x rank rows, tenant u owns rows [u*rank, (u+1)*rank)  */
  const void *a_qkv, *a_o, *a_up, *a_down;  /* bf16 [R, in]: the shrink  Z = X A^T                             */
  const void *bt_o, *bt_down;               /* bf16 [R, out]: the expand x += Zm B^T, B^T stored MN-major      */
  /* qkv / up: B lives in the last R columns of the AUGMENTED base weight layers[l].qkv_w / up_w
   * ([out, in + R], row stride in + R): [X | Zm] . [W | B]^T is one GEMM that keeps the fused bias / GELU /
   * SwiGLU epilogue.  o / down: A is STACKED under the base weight (a_o == o_w + d_model * in, same for down):
   * the backward's dX = [dY | dZ] . [W; A] is one GEMM into the bf16 activation gradient.                   */
  float *g_a_qkv, *g_a_o, *g_a_up, *g_a_down;       /* fp32 [R, in] grads (views of the flat gradient)       */
  float *g_bt_qkv, *g_bt_o, *g_bt_up, *g_bt_down;   /* fp32 [R, out]                                        */
} MaceLoraLayer;
typedef struct MaceModelDesc {
  int family;                              /* 0 llama (RMSNorm, RoPE, SwiGLU), 1 gpt2 (LayerNorm, GELU) */
  int n_layers, d_model, n_heads, n_kv_heads, head_dim, ffn, up_dim, vocab;
  float norm_eps, dpo_beta;
  const void *embed, *pos_embed, *final_norm_w, *final_norm_b;
  const MaceLayerWeights* layers;          /* [n_layers] working weights (updated in place by AdamW) */
  int n_sel; const int* sel_layers;        /* [n_sel] ascending selected (trained) layers          */
  const MaceLayerWeights* ref_layers;      /* [n_sel] frozen pi_ref copies of the selected layers  */
  const void *ref_final_norm_w, *ref_final_norm_b;  /* frozen pi_ref final norm                 */
  const MaceLayerGrads* grads;             /* [n_sel] */
  float *grad_final_norm_w, *grad_final_norm_b;
  float* grad_flat; long long n_grad;      /* zeroed by the tick before the backward               */
  const float *cos_t, *sin_t;              /* RoPE tables [max_pos][head_dim/2]                    */
  MaceKvLayout kv;
  void *k_pool, *v_pool; long long pages_per_layer;
  int* last_token;                         /* [slots] previous greedy token of each slot           */
  int* dec_counters; unsigned long long* dec_work;
  int decode_impl;                         /* see MaceAttnArgs */
  /* per-tenant LoRA (lora_R > 0): the selected layers carry adapters; their base weights (and the norms) are
   * frozen, grads are NULL except the adapters'; pi_ref = the base model (every adapter masked to zero) */
  int lora_R, lora_rank; float lora_scale;
  const MaceLoraLayer* lora;               /* [n_sel] */
  int attn_pairs;                          /* the tick's tc_items / ft_tc_items are query-block pairs (tc_pairs) */
} MaceModelDesc;
typedef struct MaceSavedActs {             /* policy activations of one selected layer (FT rows)   */
  float* x_in; void* h1; void* qkv; void* o; float* lse; float* x_mid; void* h2; void* u; void* a;
  void *zm_o, *zm_d;                       /* LoRA: masked shrink outputs of the o / down projections [n, R] bf16 */
} MaceSavedActs;
typedef struct MaceTickBuffers {           /* device scratch sized by the caller for this tick;    */
                                           /* ld_vocab: row stride (>= vocab, multiple of 8) of     */
                                           /* ft_logits, dlogits and dec_logits                     */
  float* x; void *h, *qkv, *o; float *lse, *hn; void *u, *a;   /* [T, .] ragged batch          */
  MaceSavedActs* sav;                      /* host array [n_sel]                                   */
  float *rx, *rx2, *x_lmin, *rlse; void *rh, *rqkv, *ro, *ru, *ra;  /* FT sub-batch [n_ft, .]   */
  float *dx; void* dy16; float* df; int ld_df; void *da16, *du16, *do16; float* dqkv; void* dqkv16;
  float* Dbuf;
  void* ft_h; float* ft_logits; void* dlogits; int ld_vocab; float *dh, *row_lse, *row_lp;  /* [R, .] */
  void* dec_h; float* dec_logits; int* dec_tok; float* dec_ws; size_t dec_ws_bytes;        /* [n_dec, .] */
  float *lp, *ref_lp, *loss, *margin, *coef;  /* [n_pairs][2] / [n_pairs] DPO outputs           */
  float* ws; size_t ws_bytes;              /* split-K / reduction scratch                          */
  int ld_h;                                /* row stride of h and the saved h1 / h2 (d_model + lora_R; 0 = d)   */
  float* lz; void *lzm, *ldz;              /* LoRA scratch: Z fp32 [rows, R], Zm / dZ bf16 [rows, R]            */
  int* dq_order;                           /* [n_ft * Hq] zeroed int32: deterministic dQ order (mace_attn_bwd2)  */
  unsigned long long* dec_keys;            /* [n_dec] zeroed: fused lm_head + argmax (MACE_EPI_ARGMAX); NULL = write
                                              dec_logits [n_dec, ld_vocab] and take the argmax over them          */
} MaceTickBuffers;
typedef struct MaceTickDesc {              /* device row tables of one tick (see TickBatch)        */
  int T, ft0, n_dec, R, n_pairs, need_ref; /* need_ref 0: ref_cached holds pi_ref log-probs       */
  const int *tokens, *pos, *row_seq, *row_kvi; const MaceSeq* seqs;
  const int* tc_items; int n_tc, n_tc_inference;   /* FT tiles follow the first n_tc_inference   */
  const int* dec_items; int n_dec_items;
  const int *dec_slots, *dec_rows;
  const int *ptab_slots, *ptab_rows; int n_ptab, ptab_cols;
  const int* page_copies; int n_copies;
  const int *ft_local_rows, *ft_targets, *pair_rows, *row_ps; const float* ref_cached;
  const MaceSeq* ft_seqs; const int* ft_tc_items; int n_ft_tc; const int* ft_row_seq;
  const int* bwd_items; int n_bwd;
  void** attn_events;                      /* optional cudaEvent_t[2*n_layers] around decode attention */
  void** gemm_events; int gemm_events_cap; /* optional cudaEvent_t[2*cap] around every GEMM launch     */
  long long* gemm_flops; int* gemm_count;  /* host: 2*M*N*K per instrumented GEMM, number recorded    */
  const int* row_tenant;                   /* [T] adapter (tenant) of every row; LoRA only              */
} MaceTickDesc;
int mace_model_create(mace_ctx* ctx, const MaceModelDesc* desc, mace_model** out);
int mace_model_destroy(mace_model* model);
int mace_tick_run(mace_model* model, const MaceTickBuffers* bufs, const MaceTickDesc* tick, void* stream);

/* ---------------------------------------------------------------- host bookkeeping (CPU, no GPU needed)
 * Alg. 1's packing loop (replaces the loop of schedule_iteration, scheduler.py:133-188) over the queue's first
 * n tasks in pop order with precomputed estimates mem[n] / lat[n] and is_ft[n]; more_queued: the queue holds
 * more than n. assign[i] = bin index, -1 rejected, -2 deferred, for the first out_counts[0] tasks (the
 * dequeued ones); out_counts = {dequeued, bins opened, bins examined, bin 0 n_inference, bin 0 n_ft};
 * out_bin0 = {bin 0 used MB, bin 0 max latency}. Returns 0, or 2 when the loop would dequeue past the n
 * candidates (the caller runs its own loop). */
int mace_host_alg1(int n, const double* mem, const double* lat, const int8_t* is_ft, int more_queued,
                   double budget, double hard_limit, double stop_mem, int tau_task, double lambda1, double lambda2,
                   int max_ft, int max_inf, int* assign, int* out_counts, double* out_bin0);

/* One tick's per-decode-row head statistics, capacity allocation and prune trims
 * (replaces the per-row Python of Engine._exec_decode, engine.py:496-529 -> HeadStats.update cache.py:291-309,
 * allocate_capacity cache.py:318-352, prune_decision cache.py:355-362), over per-slot state arrays:
 * ring [slots, H, W], count / pos [slots], sums / current / last_used / kept [slots, H], tau [slots] (NaN =
 * unset). Rows: slots[n] (distinct), steps[n] (decode position + 1), norms [n, H]. Writes kept_out [n, H] and
 * released_out [n]. Returns 0, or 1 without touching the state when a row hits allocate_capacity's rounding
 * corner (leftover >= H) that the caller resolves with the reference function. */
int mace_host_head_stats(int n, int H, int W, const int64_t* slots, const int64_t* steps, const double* norms,
                         double* ring, int64_t* count, int64_t* pos, double* sums, double* current,
                         double* last_used, double* tau, int64_t* kept, int c_total, double prune_window,
                         int64_t* kept_out, int64_t* released_out);

#ifdef __cplusplus
}
#endif
#endif /* MACE_B200_H */
