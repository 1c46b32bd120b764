// (3) Fused DPO loss/grad and masked AdamW — the real counterparts of the reference's fine-tune
// stand-in: Engine._exec_ft -> AlignmentEnv.ft_step (engine.py:534-536, alignment.py:168-172, where an
// FT step is `mu += ft_gain`) and the scalar DPO stage dpo_loss (alignment.py:39-47).
//
// DPO over a tick's FT pairs:
//   row stage  : per response-predicting row r: lse_r = logsumexp(logits_r), lp_r = logits_r[y_r] - lse_r
//   pair stage : lp+ = sum(chosen rows), lp- = sum(rejected rows) in fixed row order (deterministic);
//                m = (lp+ - ref+) - (lp- - ref-); loss = softplus(-beta m) (the reference's stable form);
//                dL/dlp+ = -beta sigma(-beta m) / n_pairs, dL/dlp- = -dL/dlp+
//   grad stage : dlogits_r = g_r (onehot(y_r) - softmax(logits_r)) as bf16 (input of dX = dlogits . E)
// AdamW: torch.optim.AdamW update order, every op explicitly rounded (no FMA contraction) so it is
// bit-reproducible by the fp32 restatement in oracle/adamw_ref.py; only the selected parameter
// segments are touched, then the bf16 working copy is refreshed.
#include "common.cuh"
#include "mace_internal.h"

namespace mace {

__global__ void dpo_row_kernel(const float* __restrict__ logits, int V, int ld, const int* __restrict__ targets,
                               float* __restrict__ row_lse, float* __restrict__ row_lp) {
  pdl_wait();
  pdl_trigger();
  const float* x = logits + (size_t)blockIdx.x * ld;
  __shared__ float red[32];
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < V; c += blockDim.x) mx = fmaxf(mx, x[c]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  float s = 0.f;
  for (int c = threadIdx.x; c < V; c += blockDim.x) s += __expf(x[c] - mx);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      const float lse = mx + logf(v);
      row_lse[blockIdx.x] = lse;
      row_lp[blockIdx.x] = x[targets[blockIdx.x]] - lse;
    }
  }
}

// pair_rows [n_pairs][4] = (chosen_row0, n_chosen, rejected_row0, n_rejected) in the logits rows
__global__ void dpo_pair_kernel(const float* __restrict__ row_lp, const int* __restrict__ pair_rows, int n_pairs,
                                const float* __restrict__ ref_lp, float beta, float grad_scale,
                                float* __restrict__ lp_out, float* __restrict__ loss, float* __restrict__ margin,
                                float* __restrict__ coef) {
  pdl_wait();
  pdl_trigger();
  const int p = blockIdx.x;
  const int lane = threadIdx.x;
  if (p >= n_pairs) return;
  const int* pr = pair_rows + 4 * p;
  float sums[2];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int r0 = pr[2 * side], n = pr[2 * side + 1];
    float s = 0.f;
    for (int i = lane; i < n; i += 32) s += row_lp[r0 + i];
    sums[side] = warp_sum(s);  // fixed butterfly order: deterministic
  }
  if (lane == 0) {
    lp_out[2 * p] = sums[0];
    lp_out[2 * p + 1] = sums[1];
    if (ref_lp) {
      const float m = (sums[0] - ref_lp[2 * p]) - (sums[1] - ref_lp[2 * p + 1]);
      const float x = -beta * m;  // loss = softplus(x), stable branches as alignment.py:43-47
      const float l = x > 0.f ? x + log1pf(expf(-x)) : log1pf(expf(x));
      const float sig = x > 0.f ? 1.f / (1.f + expf(-x)) : expf(x) / (1.f + expf(x));  // sigma(-beta m)
      loss[p] = l;
      margin[p] = m;
      coef[2 * p] = -beta * sig * grad_scale;
      coef[2 * p + 1] = beta * sig * grad_scale;
    }
  }
}

// dlogits[r, v] = coef[pair(r), side(r)] * (onehot(v == y_r) - exp(logit - lse_r))
__global__ void dpo_grad_kernel(const float* __restrict__ logits, int V, int ld, const int* __restrict__ targets,
                                const float* __restrict__ row_lse, const int* __restrict__ row_ps,
                                const float* __restrict__ coef, __nv_bfloat16* __restrict__ dlogits, int ldd) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.y;
  const float g = coef[row_ps[r]];
  const float lse = row_lse[r];
  const int y = targets[r];
  const float* x = logits + (size_t)r * ld;
  __nv_bfloat16* d = dlogits + (size_t)r * ldd;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) * 2; c < V; c += gridDim.x * blockDim.x * 2) {
    float v0 = -__expf(x[c] - lse) * g;
    if (c == y) v0 += g;
    if (c + 1 < V) {
      float v1 = -__expf(x[c + 1] - lse) * g;
      if (c + 1 == y) v1 += g;
      *reinterpret_cast<__nv_bfloat162*>(d + c) = __floats2bfloat162_rn(v0, v1);
    } else {
      d[c] = __float2bfloat16(v0);
    }
  }
}

// ------------------------------------------------------------------ masked AdamW
struct AdamSeg {
  const long long* offsets;  // [n_seg + 1] into the flat fp32 buffers
  __nv_bfloat16* const* weights;
  int n_seg;
};

__global__ void adamw_kernel(float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ grad, long long n, AdamSeg seg, float decay, float w1,
                             float b2, float w2, float step_size, float sbc2, float eps) {
  pdl_wait();
  pdl_trigger();
  __shared__ long long offs[65];
  for (int i = threadIdx.x; i <= seg.n_seg && i < 65; i += blockDim.x) offs[i] = seg.offsets[i];
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float g = grad[i];
    float p = __fmul_rn(master[i], decay);
    const float mm = __fadd_rn(m[i], __fmul_rn(w1, __fsub_rn(g, m[i])));
    const float vv = __fadd_rn(__fmul_rn(v[i], b2), __fmul_rn(w2, __fmul_rn(g, g)));
    const float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(vv), sbc2), eps);
    p = __fsub_rn(p, __fmul_rn(step_size, __fdiv_rn(mm, denom)));
    master[i] = p;
    m[i] = mm;
    v[i] = vv;
    int lo = 0, hi = seg.n_seg;  // find segment: offs[lo] <= i < offs[lo+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (offs[mid] <= i) lo = mid; else hi = mid;
    }
    seg.weights[lo][i - offs[lo]] = __float2bfloat16_rn(p);
  }
}

}  // namespace mace

using namespace mace;

extern "C" int mace_dpo_fused(mace_ctx* ctx, const float* logits, int R, int V, int ld, const int* targets,
                              const int* pair_rows, int n_pairs, const int* row_ps, const float* ref_lp, float beta,
                              float* row_lse, float* row_lp, float* lp_out, float* loss, float* margin, float* coef,
                              void* dlogits, int ldd, void* stream) {
  if (R <= 0 || n_pairs <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  launch_k(dpo_row_kernel, R, 1024, 0, s, logits, V, ld, targets, row_lse, row_lp);
  launch_k(dpo_pair_kernel, n_pairs, 32, 0, s, row_lp, pair_rows, n_pairs, ref_lp, beta, 1.f / n_pairs, lp_out, loss, margin,
                                         coef);
  ctx->launches += 2;
  if (dlogits && ref_lp) {
    dim3 grid((V + 2047) / 2048, R);
    launch_k(dpo_grad_kernel, grid, 1024, 0, s, logits, V, ld, targets, row_lse, row_ps, coef, (__nv_bfloat16*)dlogits, ldd);
    ctx->launches++;
  }
  return mace_check_launch(ctx, "dpo_fused");
}

extern "C" int mace_adamw_masked(mace_ctx* ctx, float* master, float* m, float* v, const float* grad, long long n,
                                 const long long* seg_offsets, void* const* seg_weights, int n_seg, float lr, float beta1,
                                 float beta2, float eps, float weight_decay, int step, void* stream) {
  if (n <= 0) return 0;
  if (n_seg > 64) return mace_fail(ctx, MACE_ERR_ARG, "adamw: at most 64 segments");
  const double bc1 = 1.0 - pow((double)beta1, step), bc2 = 1.0 - pow((double)beta2, step);
  AdamSeg seg{seg_offsets, reinterpret_cast<__nv_bfloat16* const*>(seg_weights), n_seg};
  int grid = (int)((n + 255) / 256);
  if (grid > ctx->num_sms * 8) grid = ctx->num_sms * 8;
  launch_k(adamw_kernel, grid, 256, 0, (cudaStream_t)stream, 
      master, m, v, grad, n, seg, (float)(1.0 - (double)lr * weight_decay), (float)(1.0 - (double)beta1), beta2,
      (float)(1.0 - (double)beta2), (float)((double)lr / bc1), (float)sqrt(bc2), eps);
  ctx->launches++;
  return mace_check_launch(ctx, "adamw");
}
