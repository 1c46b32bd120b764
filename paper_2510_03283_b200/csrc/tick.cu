// Native tick executor: one C call issues every launch of a hybrid tick in stream order.
//
// This is the device half of the reference's override point Engine._execute (engine.py:573-676):
// where the reference charges max(member latency) for the bin (engine.py:588-600) and advances the
// request state, the bin's ragged [prefill | decode | FT] rows run through the decoder here. The host
// loop that used to issue ~170 launches per tick from Python (ctypes + argument marshalling, ~18 us
// per launch, which left the GPU waiting on the host) is this file: the per-launch host cost drops to
// the CUDA launch itself plus two tensor-map encodes per GEMM.
//
// Order of work (one tick):
//   page-table maintenance (prompt tables, copy-on-diverge pages, decode page pops)
//   embed -> layers 0..L-1 over the shared ragged batch; from the lowest selected layer l_min on, FT
//   rows leave the shared batch and run as their own sub-batch (policy with saved activations and
//   pi_ref with the frozen copies) so both log-prob paths are kernel-for-kernel identical
//   decode head: final norm on gathered rows -> tied lm_head -> greedy argmax -> last_token scatter
//   FT: pi_ref sub-pass + DPO log-probs (or cached pi_ref), policy sub-pass + fused DPO, backward of
//   the tied lm_head (frozen), final norm and the selected layers top-down into the flat gradient.
// The masked AdamW (and the optional gradient all-reduce before it) are issued by the caller.
#include <vector>

#include "mace_internal.h"

namespace mace {

struct ModelState {
  mace_ctx* ctx;
  MaceModelDesc d;
  std::vector<MaceLayerWeights> layers, ref_layers;
  std::vector<MaceLayerGrads> grads;
  std::vector<int> sel;
  std::vector<MaceLoraLayer> lora;     // [n_sel] per-tenant adapters (LoRA mode), else empty
  const MaceTickDesc* tick = nullptr;  // the tick being issued (optional GEMM event instrumentation)
};

// activation buffers of one forward pass through a layer (FT sub-pass with save: the saved slots)
struct LayerIO {
  float* x;       // fp32 residual stream (updated in place)
  void* h1;       // attention-norm output (bf16)
  void* qkv;
  void* o;
  float* lse;     // NULL: not needed
  float* hn;      // decode head norms (last layer) or NULL
  void* h2;       // MLP-norm output
  void* u;        // up projection (pre-activation)
  void* a;        // activation
  float* x_in;    // != NULL: copy of the layer input (backward)
  float* x_mid;   // != NULL: copy of the residual after attention (backward)
  bool keep_u;    // pre-activation needed (backward): no GELU fusion
  const MaceLoraLayer* lora;  // != NULL: this layer carries the tenants' adapters (h1 / h2 rows are d + R wide)
  const int* tenant;          // LoRA: adapter of each row; NULL masks every adapter (the base model = pi_ref)
  void* zm_o;                 // LoRA: masked shrink outputs of the o / down projections [rows, R] (saved: backward)
  void* zm_d;
};

struct AttnRows {
  const MaceSeq* seqs;
  const int* tc_items;
  int n_tc;
  const int* dec_items;
  int n_dec;
  const int* row_seq;
  const int* pos;
  const int* row_kvi;
  bool paged;
};

#define MACE_TRY(expr)        \
  do {                        \
    const int rc_ = (expr);   \
    if (rc_) return rc_;      \
  } while (0)

static const size_t kBf = 2;

static int gemm(ModelState& m, const MaceTickBuffers* b, cudaStream_t s, const void* A, int lda, bool a_mn, const void* B,
                int ldb, bool b_mn, int M, int N, int K, void* out, int ldo, int mode, const void* bias,
                bool b_weights = true) {
  MaceGemmArgs g{};
  g.a = A;
  g.lda = lda;
  g.a_mn_major = a_mn;
  g.b = B;
  g.ldb = ldb;
  g.b_mn_major = b_mn;
  g.M = M;
  g.N = N;
  g.K = K;
  g.out = out;
  g.ldo = ldo;
  g.mode = mode;
  g.bias = bias;
  g.alpha = 1.f;
  g.split_k = 0;
  g.workspace = b->ws;
  g.workspace_bytes = b->ws_bytes;
  g.flags = b_weights ? MACE_GEMM_B_STATIC : 0;  // weights are only written by AdamW at the tick's end
  const MaceTickDesc* t = m.tick;
  const bool ev = t && t->gemm_events && t->gemm_count && *t->gemm_count < t->gemm_events_cap;
  if (ev) cudaEventRecord((cudaEvent_t)t->gemm_events[2 * *t->gemm_count], s);
  const int rc = mace_gemm_bf16(m.ctx, &g, s);
  if (ev) {
    cudaEventRecord((cudaEvent_t)t->gemm_events[2 * *t->gemm_count + 1], s);
    // the fused SwiGLU GEMM multiplies against both halves of the stacked [gate; up] weight
    t->gemm_flops[*t->gemm_count] = 2ll * M * N * K * (mode == MACE_EPI_BF16_SWIGLU ? 2 : 1);
    ++*t->gemm_count;
  }
  return rc;
}

// LoRA shrink of `rows` rows: Zm = bf16(scale * mask_tenant(X A_all^T)) into out (ld ldo). One GEMM for every
// tenant's block at once (N = R), then the row mask keeps each row's own tenant block (lora.cu).
static int lora_shrink(ModelState& m, const MaceTickBuffers* b, cudaStream_t s, const void* X, int ldx, const void* A,
                       int K, int rows, const int* tenant, void* out, int ldo) {
  const int R = m.d.lora_R;
  MACE_TRY(gemm(m, b, s, X, ldx, false, A, K, false, rows, R, K, b->lz, R, MACE_EPI_F32, nullptr));
  return mace_lora_mask(m.ctx, b->lz, R, tenant, rows, m.d.lora_rank, R, m.d.lora_scale, out, ldo, s);
}

static int copy(ModelState& m, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return 0;
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return mace_fail(m.ctx, MACE_ERR_CUDA, "tick: device copy failed");
  return 0;
}

static int zero(ModelState& m, void* dst, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return 0;
  if (cudaMemsetAsync(dst, 0, bytes, s) != cudaSuccess) return mace_fail(m.ctx, MACE_ERR_CUDA, "tick: memset failed");
  return 0;
}

// one decoder layer forward over rows [0, T) of `io` (engine.py:588-600 bin members, real math)
static int layer_fwd(ModelState& m, const MaceTickBuffers* b, const MaceTickDesc* t, int l, const MaceLayerWeights& W,
                     int T, const LayerIO& io, const AttnRows& ar, cudaStream_t s) {
  const MaceModelDesc& d = m.d;
  const int D = d.d_model, HO = d.n_heads * d.head_dim, QKV = (d.n_heads + 2 * d.n_kv_heads) * d.head_dim;
  const int ln = d.family == 1;
  const int R = io.lora ? d.lora_R : 0, ldh = D + R;  // LoRA: [h | Zm] rows feed the augmented qkv / up weights
  const size_t page_elems = (size_t)kPageTokens * d.head_dim;
  void* kp = ar.paged ? (void*)((char*)d.k_pool + (size_t)l * d.pages_per_layer * page_elems * kBf) : nullptr;
  void* vp = ar.paged ? (void*)((char*)d.v_pool + (size_t)l * d.pages_per_layer * page_elems * kBf) : nullptr;
  if (io.x_in) MACE_TRY(copy(m, io.x_in, io.x, (size_t)T * D * 4, s));
  MACE_TRY(mace_norm(m.ctx, io.x, D, nullptr, T, D, W.attn_norm_w, W.attn_norm_b, ln, d.norm_eps, io.h1, ldh, nullptr, s));
  if (R) MACE_TRY(lora_shrink(m, b, s, io.h1, ldh, io.lora->a_qkv, D, T, io.tenant, (char*)io.h1 + D * kBf, ldh));
  MACE_TRY(gemm(m, b, s, io.h1, ldh, false, W.qkv_w, ldh, false, T, QKV, D + R, io.qkv, QKV, MACE_EPI_BF16, W.qkv_b));
  MACE_TRY(mace_rope_kv(m.ctx, io.qkv, T, d.n_heads, d.n_kv_heads, d.head_dim, ar.pos, ar.row_seq, ar.row_kvi, ar.seqs,
                        d.cos_t, d.sin_t, d.family == 0, &d.kv, kp, vp, s));
  MaceAttnArgs a{};
  a.qkv = io.qkv;
  a.T = T;
  a.Hq = d.n_heads;
  a.Hkv = d.n_kv_heads;
  a.hd = d.head_dim;
  a.seqs = ar.seqs;
  a.kv = d.kv;
  a.k_pool = kp;
  a.v_pool = vp;
  a.pool_pages = ar.paged ? d.pages_per_layer : 0;
  a.out = io.o;
  a.lse = io.lse;
  a.head_norm = io.hn;
  a.scale = 0.f;
  a.dec_workspace = b->dec_ws;
  a.dec_workspace_bytes = b->dec_ws_bytes;
  a.dec_counters = d.dec_counters;
  a.dec_work = d.dec_work;
  a.decode_impl = d.decode_impl;
  a.tc_pairs = d.attn_pairs;
  void** ev = t->attn_events;
  if (ev && ar.n_dec > 0) {  // instrumented: tc tiles first, then the decode launch between events
    if (ar.n_tc > 0) {
      a.tc_items = ar.tc_items;
      a.n_tc = ar.n_tc;
      MACE_TRY(mace_attn_fwd(m.ctx, &a, s));
    }
    a.tc_items = nullptr;
    a.n_tc = 0;
    a.dec_items = ar.dec_items;
    a.n_dec = ar.n_dec;
    cudaEventRecord((cudaEvent_t)ev[2 * l], s);
    MACE_TRY(mace_attn_fwd(m.ctx, &a, s));
    cudaEventRecord((cudaEvent_t)ev[2 * l + 1], s);
  } else {
    a.tc_items = ar.tc_items;
    a.n_tc = ar.n_tc;
    a.dec_items = ar.dec_items;
    a.n_dec = ar.n_dec;
    MACE_TRY(mace_attn_fwd(m.ctx, &a, s));
  }
  MACE_TRY(gemm(m, b, s, io.o, HO, false, W.o_w, HO, false, T, D, HO, io.x, D, MACE_EPI_F32_ADD, W.o_b));
  if (R) {  // x += Zm_o B_o^T (B^T [R, D] read MN-major)
    MACE_TRY(lora_shrink(m, b, s, io.o, HO, io.lora->a_o, HO, T, io.tenant, io.zm_o, R));
    MACE_TRY(gemm(m, b, s, io.zm_o, R, false, io.lora->bt_o, D, true, T, D, R, io.x, D, MACE_EPI_F32_ADD, nullptr));
  }
  if (io.x_mid) MACE_TRY(copy(m, io.x_mid, io.x, (size_t)T * D * 4, s));
  MACE_TRY(mace_norm(m.ctx, io.x, D, nullptr, T, D, W.mlp_norm_w, W.mlp_norm_b, ln, d.norm_eps, io.h2, ldh, nullptr, s));
  if (R) MACE_TRY(lora_shrink(m, b, s, io.h2, ldh, io.lora->a_up, D, T, io.tenant, (char*)io.h2 + D * kBf, ldh));
  if (ln && !io.keep_u) {  // GPT-2: GELU fused into the up-projection epilogue
    MACE_TRY(gemm(m, b, s, io.h2, ldh, false, W.up_w, ldh, false, T, d.ffn, D + R, io.a, d.ffn, MACE_EPI_BF16_GELU, W.up_b));
  } else if (!ln && !io.keep_u) {  // Llama: SwiGLU fused (gate / up halves of one accumulator tile)
    MACE_TRY(gemm(m, b, s, io.h2, ldh, false, W.up_w, ldh, false, T, d.ffn, D + R, io.a, d.ffn, MACE_EPI_BF16_SWIGLU,
                  nullptr));
  } else {
    MACE_TRY(gemm(m, b, s, io.h2, ldh, false, W.up_w, ldh, false, T, d.up_dim, D + R, io.u, d.up_dim, MACE_EPI_BF16,
                  W.up_b));
    MACE_TRY(mace_act(m.ctx, io.u, T, d.ffn, d.family == 0, io.a, s));
  }
  MACE_TRY(gemm(m, b, s, io.a, d.ffn, false, W.down_w, d.ffn, false, T, D, d.ffn, io.x, D, MACE_EPI_F32_ADD, W.down_b));
  if (R) {
    MACE_TRY(lora_shrink(m, b, s, io.a, d.ffn, io.lora->a_down, d.ffn, T, io.tenant, io.zm_d, R));
    MACE_TRY(gemm(m, b, s, io.zm_d, R, false, io.lora->bt_down, D, true, T, D, R, io.x, D, MACE_EPI_F32_ADD, nullptr));
  }
  return 0;
}

// FT sub-batch through the selected layers from the shared l_min input, then final norm + lm_head on
// the response-predicting rows (logits into ft_logits)
static int sub_pass(ModelState& m, const MaceTickBuffers* b, const MaceTickDesc* t, bool policy, float* x, cudaStream_t s) {
  const MaceModelDesc& d = m.d;
  const int n = t->T - t->ft0, D = d.d_model;
  MACE_TRY(copy(m, x, b->x_lmin, (size_t)n * D * 4, s));
  AttnRows ar{t->ft_seqs, t->ft_tc_items, t->n_ft_tc, nullptr, 0, t->ft_row_seq, t->pos + t->ft0, nullptr, false};
  for (size_t i = 0; i < m.sel.size(); ++i) {
    LayerIO io{};
    io.x = x;
    if (!m.lora.empty()) {  // pi_ref = the base model: every adapter masked (tenant NULL), same kernels
      io.lora = &m.lora[i];
      io.tenant = policy && t->row_tenant ? t->row_tenant + t->ft0 : nullptr;
      io.zm_o = policy ? b->sav[i].zm_o : b->lzm;
      io.zm_d = policy ? b->sav[i].zm_d : b->lzm;
    }
    if (policy) {
      const MaceSavedActs& sv = b->sav[i];
      io.h1 = sv.h1;
      io.qkv = sv.qkv;
      io.o = sv.o;
      io.lse = sv.lse;
      io.h2 = sv.h2;
      io.u = sv.u;
      io.a = sv.a;
      io.x_in = sv.x_in;
      io.x_mid = sv.x_mid;
      io.keep_u = true;
    } else {
      io.h1 = io.h2 = b->rh;
      io.qkv = b->rqkv;
      io.o = b->ro;
      io.u = b->ru;
      io.a = b->ra;
      io.keep_u = true;  // same activation path as the policy pass: margin exactly 0 while pi_theta = pi_ref
    }
    MACE_TRY(layer_fwd(m, b, t, m.sel[i], policy ? m.layers[m.sel[i]] : m.ref_layers[i], n, io, ar, s));
  }
  const void* fw = policy ? d.final_norm_w : d.ref_final_norm_w;
  const void* fb = policy ? d.final_norm_b : d.ref_final_norm_b;
  MACE_TRY(mace_norm(m.ctx, x, D, t->ft_local_rows, t->R, D, fw, fb, d.family == 1, d.norm_eps, b->ft_h, D, nullptr, s));
  MACE_TRY(gemm(m, b, s, b->ft_h, D, false, d.embed, D, false, t->R, d.vocab, D, b->ft_logits, b->ld_vocab,
                MACE_EPI_F32, nullptr));
  return 0;
}

static int colsum(ModelState& m, const MaceTickBuffers* b, const void* y16, int n, int N, float* out, cudaStream_t s) {
  if (!out) return 0;
  return mace_colsum_bf16(m.ctx, y16, n, N, N, out, b->ws, b->ws_bytes, s);
}

// LoRA layer backward (base weights and norms frozen): dx -> grad wrt the layer input; the adapters' dA / dB^T into
// the flat gradient. Per projection with input X, Zm = s * mask(X A^T), Y = X W^T + Zm B^T:
//   dB^T += Zm^T dY,  dZ = s * mask(dY B),  dA += dZ^T X,  dX = dY W + dZ A
// o / down: dY goes to the first d columns of dy16 ([n, d + R]) and dZ to the last R, so [dY | dZ] . [W; A] (A stacked
// under W) is one GEMM into the bf16 dX; qkv / up: [dX | dZm] = dY . [W | B] is one GEMM, then dX += dZ A.
static int layer_bwd_lora(ModelState& m, const MaceTickBuffers* b, const MaceTickDesc* t, int i, cudaStream_t s) {
  const MaceModelDesc& d = m.d;
  const int l = m.sel[i];
  const MaceLayerWeights& W = m.layers[l];
  const MaceLoraLayer& lo = m.lora[i];
  const MaceSavedActs& sv = b->sav[i];
  const int n = t->T - t->ft0, D = d.d_model, F = d.ffn, UP = d.up_dim, R = d.lora_R, rk = d.lora_rank;
  const int HO = d.n_heads * d.head_dim, QKV = (d.n_heads + 2 * d.n_kv_heads) * d.head_dim;
  const int ln = d.family == 1, ldh = D + R, ldy = D + R;
  const float sc = d.lora_scale;
  const int* ten = t->row_tenant ? t->row_tenant + t->ft0 : nullptr;
  void* dz_y = (char*)b->dy16 + D * kBf;  // last R columns of [dY | dZ]
  // MLP down
  MACE_TRY(mace_f32_to_bf16_2d(m.ctx, b->dx, D, n, D, b->dy16, ldy, s));
  MACE_TRY(gemm(m, b, s, b->dy16, ldy, false, lo.bt_down, D, false, n, R, D, b->lz, R, MACE_EPI_F32, nullptr));
  MACE_TRY(mace_lora_mask(m.ctx, b->lz, R, ten, n, rk, R, sc, dz_y, ldy, s));
  MACE_TRY(gemm(m, b, s, sv.zm_d, R, true, b->dy16, ldy, true, R, D, n, lo.g_bt_down, D, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(gemm(m, b, s, dz_y, ldy, true, sv.a, F, true, R, F, n, lo.g_a_down, F, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(gemm(m, b, s, b->dy16, ldy, false, W.down_w, F, true, n, F, D + R, b->da16, F, MACE_EPI_BF16, nullptr));
  MACE_TRY(mace_act_bwd(m.ctx, sv.u, b->da16, n, F, d.family == 0, b->du16, s));
  // MLP up (augmented)
  MACE_TRY(gemm(m, b, s, (char*)sv.h2 + D * kBf, ldh, true, b->du16, UP, true, R, UP, n, lo.g_bt_up, UP, MACE_EPI_F32_ADD,
                nullptr, false));
  MACE_TRY(gemm(m, b, s, b->du16, UP, false, W.up_w, ldh, true, n, D + R, UP, b->df, b->ld_df, MACE_EPI_F32, nullptr));
  MACE_TRY(mace_lora_mask(m.ctx, b->df + D, b->ld_df, ten, n, rk, R, sc, b->ldz, R, s));
  MACE_TRY(gemm(m, b, s, b->ldz, R, true, sv.h2, ldh, true, R, D, n, lo.g_a_up, D, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(gemm(m, b, s, b->ldz, R, false, lo.a_up, D, true, n, D, R, b->df, b->ld_df, MACE_EPI_F32_ADD, nullptr));
  MACE_TRY(mace_norm_bwd(m.ctx, sv.x_mid, D, nullptr, b->df, b->ld_df, n, D, W.mlp_norm_w, ln, d.norm_eps, b->dx, D,
                         nullptr, nullptr, nullptr, b->ws, b->ws_bytes, s));
  // attention: o projection
  MACE_TRY(mace_f32_to_bf16_2d(m.ctx, b->dx, D, n, D, b->dy16, ldy, s));
  MACE_TRY(gemm(m, b, s, b->dy16, ldy, false, lo.bt_o, D, false, n, R, D, b->lz, R, MACE_EPI_F32, nullptr));
  MACE_TRY(mace_lora_mask(m.ctx, b->lz, R, ten, n, rk, R, sc, dz_y, ldy, s));
  MACE_TRY(gemm(m, b, s, sv.zm_o, R, true, b->dy16, ldy, true, R, D, n, lo.g_bt_o, D, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(gemm(m, b, s, dz_y, ldy, true, sv.o, HO, true, R, HO, n, lo.g_a_o, HO, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(gemm(m, b, s, b->dy16, ldy, false, W.o_w, HO, true, n, HO, D + R, b->do16, HO, MACE_EPI_BF16, nullptr));
  // attention core (dense causal FT sequences)
  MACE_TRY(zero(m, b->dqkv, (size_t)n * QKV * 4, s));
  MACE_TRY(mace_attn_bwd2(m.ctx, sv.qkv, sv.o, b->do16, sv.lse, n, d.n_heads, d.n_kv_heads, d.head_dim, t->ft_seqs,
                          t->bwd_items, t->n_bwd, 0, b->Dbuf, b->dqkv, b->dq_order, s));
  if (d.family == 0)
    MACE_TRY(mace_rope_bwd(m.ctx, b->dqkv, n, d.n_heads, d.n_kv_heads, d.head_dim, t->pos + t->ft0, d.cos_t, d.sin_t, s));
  MACE_TRY(mace_f32_to_bf16(m.ctx, b->dqkv, (long long)n * QKV, b->dqkv16, s));
  // qkv (augmented)
  MACE_TRY(gemm(m, b, s, (char*)sv.h1 + D * kBf, ldh, true, b->dqkv16, QKV, true, R, QKV, n, lo.g_bt_qkv, QKV,
                MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(gemm(m, b, s, b->dqkv16, QKV, false, W.qkv_w, ldh, true, n, D + R, QKV, b->df, b->ld_df, MACE_EPI_F32, nullptr));
  MACE_TRY(mace_lora_mask(m.ctx, b->df + D, b->ld_df, ten, n, rk, R, sc, b->ldz, R, s));
  MACE_TRY(gemm(m, b, s, b->ldz, R, true, sv.h1, ldh, true, R, D, n, lo.g_a_qkv, D, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(gemm(m, b, s, b->ldz, R, false, lo.a_qkv, D, true, n, D, R, b->df, b->ld_df, MACE_EPI_F32_ADD, nullptr));
  MACE_TRY(mace_norm_bwd(m.ctx, sv.x_in, D, nullptr, b->df, b->ld_df, n, D, W.attn_norm_w, ln, d.norm_eps, b->dx, D,
                         nullptr, nullptr, nullptr, b->ws, b->ws_bytes, s));
  return 0;
}

// dx (grad wrt the layer output, FT rows) -> grad wrt its input; dW of the layer into the flat grad
static int layer_bwd(ModelState& m, const MaceTickBuffers* b, const MaceTickDesc* t, int i, cudaStream_t s) {
  if (!m.lora.empty()) return layer_bwd_lora(m, b, t, i, s);
  const MaceModelDesc& d = m.d;
  const int l = m.sel[i];
  const MaceLayerWeights& W = m.layers[l];
  const MaceLayerGrads& g = m.grads[i];
  const MaceSavedActs& sv = b->sav[i];
  const int n = t->T - t->ft0, D = d.d_model, F = d.ffn, UP = d.up_dim;
  const int HO = d.n_heads * d.head_dim, QKV = (d.n_heads + 2 * d.n_kv_heads) * d.head_dim;
  const int ln = d.family == 1;
  // MLP down: dW = dy^T a, db = colsum(dy), da = dy W
  MACE_TRY(mace_f32_to_bf16(m.ctx, b->dx, (long long)n * D, b->dy16, s));
  MACE_TRY(gemm(m, b, s, b->dy16, D, true, sv.a, F, true, D, F, n, g.down_w, F, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(colsum(m, b, b->dy16, n, D, g.down_b, s));
  MACE_TRY(gemm(m, b, s, b->dy16, D, false, W.down_w, F, true, n, F, D, b->da16, F, MACE_EPI_BF16, nullptr));
  MACE_TRY(mace_act_bwd(m.ctx, sv.u, b->da16, n, F, d.family == 0, b->du16, s));
  // MLP up
  MACE_TRY(gemm(m, b, s, b->du16, UP, true, sv.h2, D, true, UP, D, n, g.up_w, D, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(colsum(m, b, b->du16, n, UP, g.up_b, s));
  MACE_TRY(gemm(m, b, s, b->du16, UP, false, W.up_w, D, true, n, D, UP, b->df, b->ld_df, MACE_EPI_F32, nullptr));
  MACE_TRY(mace_norm_bwd(m.ctx, sv.x_mid, D, nullptr, b->df, b->ld_df, n, D, W.mlp_norm_w, ln, d.norm_eps, b->dx, D,
                         nullptr, g.mlp_norm_w, g.mlp_norm_b, b->ws, b->ws_bytes, s));
  // attention: o projection
  MACE_TRY(mace_f32_to_bf16(m.ctx, b->dx, (long long)n * D, b->dy16, s));
  MACE_TRY(gemm(m, b, s, b->dy16, D, true, sv.o, HO, true, D, HO, n, g.o_w, HO, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(colsum(m, b, b->dy16, n, D, g.o_b, s));
  MACE_TRY(gemm(m, b, s, b->dy16, D, false, W.o_w, HO, true, n, HO, D, b->do16, HO, MACE_EPI_BF16, nullptr));
  // attention core (dense causal FT sequences)
  MACE_TRY(zero(m, b->dqkv, (size_t)n * QKV * 4, s));
  MACE_TRY(mace_attn_bwd2(m.ctx, sv.qkv, sv.o, b->do16, sv.lse, n, d.n_heads, d.n_kv_heads, d.head_dim, t->ft_seqs,
                          t->bwd_items, t->n_bwd, 0, b->Dbuf, b->dqkv, b->dq_order, s));
  if (d.family == 0)
    MACE_TRY(mace_rope_bwd(m.ctx, b->dqkv, n, d.n_heads, d.n_kv_heads, d.head_dim, t->pos + t->ft0, d.cos_t, d.sin_t, s));
  MACE_TRY(mace_f32_to_bf16(m.ctx, b->dqkv, (long long)n * QKV, b->dqkv16, s));
  MACE_TRY(gemm(m, b, s, b->dqkv16, QKV, true, sv.h1, D, true, QKV, D, n, g.qkv_w, D, MACE_EPI_F32_ADD, nullptr, false));
  MACE_TRY(colsum(m, b, b->dqkv16, n, QKV, g.qkv_b, s));
  MACE_TRY(gemm(m, b, s, b->dqkv16, QKV, false, W.qkv_w, D, true, n, D, QKV, b->df, b->ld_df, MACE_EPI_F32, nullptr));
  MACE_TRY(mace_norm_bwd(m.ctx, sv.x_in, D, nullptr, b->df, b->ld_df, n, D, W.attn_norm_w, ln, d.norm_eps, b->dx, D,
                         nullptr, g.attn_norm_w, g.attn_norm_b, b->ws, b->ws_bytes, s));
  return 0;
}

static int ft_step(ModelState& m, const MaceTickBuffers* b, const MaceTickDesc* t, cudaStream_t s) {
  const MaceModelDesc& d = m.d;
  const int n = t->T - t->ft0, D = d.d_model, R = t->R, P = t->n_pairs;
  if (t->need_ref) {
    MACE_TRY(sub_pass(m, b, t, false, b->rx2, s));
    MACE_TRY(mace_dpo_fused(m.ctx, b->ft_logits, R, d.vocab, b->ld_vocab, t->ft_targets, t->pair_rows, P, t->row_ps, nullptr,
                            0.f, b->row_lse, b->row_lp, b->ref_lp, nullptr, nullptr, nullptr, nullptr, 0, s));
  } else {
    MACE_TRY(copy(m, b->ref_lp, t->ref_cached, (size_t)P * 2 * 4, s));
  }
  MACE_TRY(sub_pass(m, b, t, true, b->rx, s));
  MACE_TRY(mace_dpo_fused(m.ctx, b->ft_logits, R, d.vocab, b->ld_vocab, t->ft_targets, t->pair_rows, P, t->row_ps, b->ref_lp,
                          d.dpo_beta, b->row_lse, b->row_lp, b->lp, b->loss, b->margin, b->coef, b->dlogits,
                          b->ld_vocab, s));
  // backward: tied lm_head (frozen) -> final norm -> selected layers top-down
  MACE_TRY(zero(m, d.grad_flat, (size_t)d.n_grad * 4, s));
  MACE_TRY(gemm(m, b, s, b->dlogits, b->ld_vocab, false, d.embed, D, true, R, D, d.vocab, b->dh, D, MACE_EPI_F32,
                nullptr));
  MACE_TRY(zero(m, b->dx, (size_t)n * D * 4, s));
  MACE_TRY(mace_norm_bwd(m.ctx, b->rx, D, t->ft_local_rows, b->dh, D, R, D, d.final_norm_w, d.family == 1, d.norm_eps,
                         b->dx, D, t->ft_local_rows, d.grad_final_norm_w, d.grad_final_norm_b, b->ws, b->ws_bytes, s));
  for (int i = (int)m.sel.size() - 1; i >= 0; --i) MACE_TRY(layer_bwd(m, b, t, i, s));
  return 0;
}

static int tick_run(ModelState& m, const MaceTickBuffers* b, const MaceTickDesc* t, cudaStream_t s) {
  const MaceModelDesc& d = m.d;
  mace_ctx* ctx = m.ctx;
  // ---- page-table maintenance (host page-manager decisions -> device)
  if (t->n_ptab > 0)
    MACE_TRY(mace_kv_set_prompt_tables(ctx, &d.kv, t->ptab_slots, t->ptab_rows, t->n_ptab, t->ptab_cols, s));
  if (t->n_copies > 0)
    MACE_TRY(mace_kv_page_copy(ctx, t->page_copies, t->n_copies, d.n_kv_heads, d.head_dim, d.pages_per_layer, d.n_layers,
                               d.k_pool, d.v_pool, s));
  if (t->n_dec > 0) MACE_TRY(mace_kv_decode_alloc(ctx, &d.kv, t->dec_slots, t->n_dec, s));
  const int T = t->T, ft0 = t->ft0, n_ft = T - ft0, D = d.d_model;
  if (T == 0) return 0;
  // ---- forward through all layers (one ragged batch)
  MACE_TRY(mace_embed(ctx, t->tokens, t->pos, d.last_token, d.embed, d.pos_embed, T, D, b->x, s));
  const bool has_ft = n_ft > 0 && t->n_pairs > 0;
  const int l_min = m.sel.empty() ? d.n_layers : m.sel[0];
  const int l_sel0 = l_min;  // LoRA: the selected layers are contiguous (the top n_sel), adapter i = layer l_sel0 + i
  for (int l = 0; l < d.n_layers; ++l) {
    const bool top = has_ft && l >= l_min;
    const int T_l = top ? ft0 : T;
    if (has_ft && l == l_min) MACE_TRY(copy(m, b->x_lmin, b->x + (size_t)ft0 * D, (size_t)n_ft * D * 4, s));
    if (T_l == 0) continue;
    AttnRows ar{t->seqs, t->tc_items, top ? t->n_tc_inference : t->n_tc, t->dec_items, t->n_dec_items,
                t->row_seq, t->pos, t->row_kvi, true};
    LayerIO io{};
    io.x = b->x;
    io.h1 = io.h2 = b->h;
    io.qkv = b->qkv;
    io.o = b->o;
    io.hn = l == d.n_layers - 1 ? b->hn : nullptr;
    io.u = b->u;
    io.a = b->a;
    if (!m.lora.empty() && l >= l_sel0) {  // a selected layer: every row runs with its own tenant's adapter
      io.lora = &m.lora[l - l_sel0];
      io.tenant = t->row_tenant;
      io.zm_o = io.zm_d = b->lzm;
    }
    MACE_TRY(layer_fwd(m, b, t, l, m.layers[l], T_l, io, ar, s));
  }
  // ---- decode rows: final norm on gathered rows -> lm_head -> greedy token -> last_token
  if (t->n_dec > 0) {
    MACE_TRY(mace_norm(ctx, b->x, D, t->dec_rows, t->n_dec, D, d.final_norm_w, d.final_norm_b, d.family == 1, d.norm_eps,
                       b->dec_h, D, nullptr, s));
    if (b->dec_keys) {  // fused: the lm_head epilogue reduces every row to its argmax key, no [n_dec, V] logits
      MACE_TRY(gemm(m, b, s, b->dec_h, D, false, d.embed, D, false, t->n_dec, d.vocab, D, b->dec_keys, 0,
                    MACE_EPI_ARGMAX, nullptr));
      MACE_TRY(mace_argmax_keys(ctx, b->dec_keys, t->n_dec, b->dec_tok, s));
    } else {            // logits kept for the caller (oracle replays read them)
      MACE_TRY(gemm(m, b, s, b->dec_h, D, false, d.embed, D, false, t->n_dec, d.vocab, D, b->dec_logits, b->ld_vocab,
                    MACE_EPI_F32, nullptr));
      MACE_TRY(mace_argmax(ctx, b->dec_logits, t->n_dec, d.vocab, b->ld_vocab, b->dec_tok, s));
    }
    MACE_TRY(mace_scatter_tokens(ctx, b->dec_tok, t->dec_slots, t->n_dec, d.last_token, s));
  }
  if (has_ft) MACE_TRY(ft_step(m, b, t, s));
  return mace_check_launch(ctx, "tick");
}

}  // namespace mace

using namespace mace;

struct mace_model : public mace::ModelState {};

extern "C" int mace_model_create(mace_ctx* ctx, const MaceModelDesc* desc, mace_model** out) {
  if (!ctx || !desc || !out) return MACE_ERR_ARG;
  *out = nullptr;
  if (desc->family != 0 && desc->family != 1) return mace_fail(ctx, MACE_ERR_ARG, "model: family must be 0 or 1");
  if (desc->n_layers <= 0 || !desc->layers) return mace_fail(ctx, MACE_ERR_ARG, "model: no layers");
  if (desc->n_sel < 0 || desc->n_sel > desc->n_layers || (desc->n_sel && (!desc->sel_layers || !desc->ref_layers ||
                                                                          !desc->grads)))
    return mace_fail(ctx, MACE_ERR_ARG, "model: bad selected-layer tables");
  mace_model* m = new mace_model();
  m->ctx = ctx;
  m->d = *desc;
  m->layers.assign(desc->layers, desc->layers + desc->n_layers);
  m->sel.assign(desc->sel_layers, desc->sel_layers + desc->n_sel);
  m->ref_layers.assign(desc->ref_layers, desc->ref_layers + desc->n_sel);
  m->grads.assign(desc->grads, desc->grads + desc->n_sel);
  for (size_t i = 1; i < m->sel.size(); ++i) {
    if (m->sel[i] <= m->sel[i - 1]) {
      delete m;
      return mace_fail(ctx, MACE_ERR_ARG, "model: selected layers must be ascending");
    }
  }
  if (desc->lora_R > 0) {
    const int D = desc->d_model, HO = desc->n_heads * desc->head_dim;
    const char* why = nullptr;
    if (!desc->lora || desc->lora_rank <= 0 || desc->lora_R % 8 || desc->lora_R % desc->lora_rank)
      why = "model: LoRA needs adapters, rank > 0 and R = tenants x rank with R % 8 == 0";
    for (size_t i = 0; !why && i < m->sel.size(); ++i) {
      if (i && m->sel[i] != m->sel[i - 1] + 1) why = "model: LoRA layers must be contiguous";
      const MaceLayerWeights& W = desc->layers[m->sel[i]];
      const MaceLoraLayer& lo = desc->lora[i];
      if (lo.a_o != (const char*)W.o_w + (size_t)D * HO * 2 || lo.a_down != (const char*)W.down_w + (size_t)D * desc->ffn * 2)
        why = "model: LoRA a_o / a_down must be stacked directly under o_w / down_w";
    }
    if (why) {
      delete m;
      return mace_fail(ctx, MACE_ERR_ARG, why);
    }
    m->lora.assign(desc->lora, desc->lora + desc->n_sel);
  }
  m->d.lora = nullptr;
  m->d.layers = nullptr;  // the copies above own the tables
  m->d.sel_layers = nullptr;
  m->d.ref_layers = nullptr;
  m->d.grads = nullptr;
  *out = m;
  return MACE_OK;
}

extern "C" int mace_model_destroy(mace_model* model) {
  delete model;
  return MACE_OK;
}

extern "C" int mace_tick_run(mace_model* model, const MaceTickBuffers* bufs, const MaceTickDesc* tick, void* stream) {
  if (!model || !bufs || !tick) return MACE_ERR_ARG;
  if (tick->T > 0 && (!bufs->x || !bufs->h || !bufs->qkv || !bufs->o || !bufs->ws))
    return mace_fail(model->ctx, MACE_ERR_ARG, "tick: missing activation buffers");
  if (tick->T - tick->ft0 > 0 && tick->n_pairs > 0 && !bufs->sav && model->sel.size())
    return mace_fail(model->ctx, MACE_ERR_ARG, "tick: FT rows need saved-activation buffers");
  if (!model->lora.empty() && (!bufs->lz || !bufs->lzm || bufs->ld_h != model->d.d_model + model->d.lora_R ||
                               (tick->T - tick->ft0 > 0 && (!bufs->ldz || !tick->row_tenant))))
    return mace_fail(model->ctx, MACE_ERR_ARG, "tick: LoRA needs lz / lzm / ldz scratch, ld_h = d + R and row tenants");
  model->tick = tick;
  const int rc = tick_run(*model, bufs, tick, (cudaStream_t)stream);
  model->tick = nullptr;
  return rc;
}
