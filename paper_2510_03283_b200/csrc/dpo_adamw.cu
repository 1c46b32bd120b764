// (3) Fused DPO loss/grad and masked AdamW — the real counterparts of the reference's fine-tune
// stand-in: Engine._exec_ft -> AlignmentEnv.ft_step (engine.py:534-536, alignment.py:168-172, where an
// FT step is `mu += ft_gain`) and the scalar DPO stage dpo_loss (alignment.py:39-47).
//
// DPO over a tick's FT pairs:
//   row stage  : per response-predicting row r: lse_r = logsumexp(logits_r), lp_r = logits_r[y_r] - lse_r
//   pair stage : lp+ = sum(chosen rows), lp- = sum(rejected rows) in fixed row order (deterministic);
//                m = (lp+ - ref+) - (lp- - ref-); loss = softplus(-beta m): the reference's dpo_loss in fp64,
//                same branches and expression order (dpo_scalar below, pinned to tests/golden/dpo_golden.json);
//                dL/dlp+ = -beta sigma(-beta m) / n_pairs, dL/dlp- = -dL/dlp+
//   grad stage : dlogits_r = g_r (onehot(y_r) - softmax(logits_r)) as bf16 (input of dX = dlogits . E)
// AdamW: torch.optim.AdamW update order, every op explicitly rounded (no FMA contraction) so it is
// bit-reproducible by the numpy fp32 restatement in tests/test_dpo_adamw_gpu.py; only the selected parameter
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

// The reference's scalar stage, dpo_loss (alignment.py:39-47), in IEEE fp64 with its exact expression order:
//   margin = delta_plus - delta_minus;  x = -beta * margin;  loss = x > 0 ? x + log1p(exp(-x)) : log1p(exp(x))
// plus sigma(-beta m) = dL/d(-beta m) for the gradient, from the same x. Shared by the fused DPO pair stage
// and mace_dpo_scalar (the entry point the golden-vector test drives with the reference's own inputs).
__device__ __forceinline__ void dpo_scalar(double delta_plus, double delta_minus, double beta, double& margin,
                                           double& loss, double& sig) {
  margin = delta_plus - delta_minus;
  const double x = -beta * margin;
  if (x > 0.0) {
    loss = x + log1p(exp(-x));
    sig = 1.0 / (1.0 + exp(-x));
  } else {
    const double e = exp(x);
    loss = log1p(e);
    sig = e / (1.0 + e);
  }
}

__global__ void dpo_scalar_kernel(const double* __restrict__ dplus, const double* __restrict__ dminus,
                                  const double* __restrict__ beta, int n, double* __restrict__ loss,
                                  double* __restrict__ margin, double* __restrict__ sig) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double m, l, sg;
  dpo_scalar(dplus[i], dminus[i], beta[i], m, l, sg);
  loss[i] = l;
  if (margin) margin[i] = m;
  if (sig) sig[i] = sg;
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
      // delta_plus = lp+ - ref+, delta_minus = lp- - ref- (the reference's MarginSample, alignment.py:30-37);
      // the scalar stage in fp64 exactly as dpo_loss (alignment.py:39-47)
      double m, l, sig;
      dpo_scalar((double)sums[0] - (double)ref_lp[2 * p], (double)sums[1] - (double)ref_lp[2 * p + 1], (double)beta,
                 m, l, sig);
      loss[p] = (float)l;
      margin[p] = (float)m;
      coef[2 * p] = (float)(-(double)beta * sig * (double)grad_scale);
      coef[2 * p + 1] = (float)((double)beta * sig * (double)grad_scale);
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

// one element of torch.optim.AdamW (decoupled weight decay; single-tensor order), every op rounded explicitly
// (no FMA contraction) so the numpy fp32 restatement in tests reproduces it bit for bit
__device__ __forceinline__ void adamw_elem(float& p, float& mm, float& vv, float g, float decay, float w1, float b2,
                                           float w2, float step_size, float sbc2, float eps) {
  p = __fmul_rn(p, decay);
  mm = __fadd_rn(mm, __fmul_rn(w1, __fsub_rn(g, mm)));
  vv = __fadd_rn(__fmul_rn(vv, b2), __fmul_rn(w2, __fmul_rn(g, g)));
  const float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(vv), sbc2), eps);
  p = __fsub_rn(p, __fmul_rn(step_size, __fdiv_rn(mm, denom)));
}

__device__ __forceinline__ int seg_of(const long long* offs, int n_seg, long long i) {
  int lo = 0, hi = n_seg;  // offs[lo] <= i < offs[lo+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (offs[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// Vector path (every segment offset a multiple of 4, every bf16 copy 8-byte aligned): one float4 of each fp32
// stream per step, two steps per thread in flight, streaming (evict-first) loads and stores -- each byte is
// touched once, 30 B per parameter (master, m, v r/w 24 B, grad r 4 B, bf16 w 2 B).
__global__ void __launch_bounds__(256) adamw_vec_kernel(float4* __restrict__ master, float4* __restrict__ m,
                                                        float4* __restrict__ v, const float4* __restrict__ grad,
                                                        long long n4, AdamSeg seg, float decay, float w1, float b2,
                                                        float w2, float step_size, float sbc2, float eps) {
  pdl_wait();
  pdl_trigger();
  __shared__ long long offs[65];
  for (int i = threadIdx.x; i <= seg.n_seg && i < 65; i += blockDim.x) offs[i] = seg.offsets[i];
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long q0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; q0 < n4; q0 += 2 * stride) {
    float4 P[2], M[2], V[2], G[2];
    long long qs[2] = {q0, q0 + stride};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (qs[u] < n4) {
        P[u] = __ldcs(master + qs[u]);
        M[u] = __ldcs(m + qs[u]);
        V[u] = __ldcs(v + qs[u]);
        G[u] = __ldcs(grad + qs[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (qs[u] >= n4) continue;
      float4 p = P[u], mm = M[u], vv = V[u];
      const float4 g = G[u];
      adamw_elem(p.x, mm.x, vv.x, g.x, decay, w1, b2, w2, step_size, sbc2, eps);
      adamw_elem(p.y, mm.y, vv.y, g.y, decay, w1, b2, w2, step_size, sbc2, eps);
      adamw_elem(p.z, mm.z, vv.z, g.z, decay, w1, b2, w2, step_size, sbc2, eps);
      adamw_elem(p.w, mm.w, vv.w, g.w, decay, w1, b2, w2, step_size, sbc2, eps);
      __stcs(master + qs[u], p);
      __stcs(m + qs[u], mm);
      __stcs(v + qs[u], vv);
      const long long i = 4 * qs[u];
      const int sg = seg_of(offs, seg.n_seg, i);
      __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y), hi = __floats2bfloat162_rn(p.z, p.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(seg.weights[sg] + (i - offs[sg])) = pk;
    }
  }
}

// Sparse segments (per-tenant adapters): virtual index v in [0, n) -> segment s (vstart[s] <= v < vstart[s+1]) ->
// flat element flat[s] + (v - vstart[s]). VEC: every vstart / flat offset a multiple of 4, float4 streams.
struct AdamSparse {
  const long long* vstart;  // [n_seg + 1]
  const long long* flat;    // [n_seg]
  __nv_bfloat16* const* weights;
  int n_seg;
};

template <bool VEC>
__global__ void __launch_bounds__(256) adamw_sparse_kernel(float* __restrict__ master, float* __restrict__ m,
                                                           float* __restrict__ v, const float* __restrict__ grad,
                                                           long long n, AdamSparse sg, float decay, float w1, float b2,
                                                           float w2, float step_size, float sbc2, float eps) {
  pdl_wait();
  pdl_trigger();
  __shared__ long long vs[65], fl[64];
  for (int i = threadIdx.x; i <= sg.n_seg && i < 65; i += blockDim.x) {
    vs[i] = sg.vstart[i];
    if (i < sg.n_seg) fl[i] = sg.flat[i];
  }
  __syncthreads();
  const int W = VEC ? 4 : 1;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q * W < n; q += (long long)gridDim.x * blockDim.x) {
    const long long vi = q * W;
    const int s = seg_of(vs, sg.n_seg, vi);
    const long long f = fl[s] + (vi - vs[s]);
    __nv_bfloat16* wp = sg.weights[s] + (vi - vs[s]);
    if (VEC) {
      float4 p = *reinterpret_cast<float4*>(master + f), mm = *reinterpret_cast<float4*>(m + f),
             vv = *reinterpret_cast<float4*>(v + f);
      const float4 g = *reinterpret_cast<const float4*>(grad + f);
      adamw_elem(p.x, mm.x, vv.x, g.x, decay, w1, b2, w2, step_size, sbc2, eps);
      adamw_elem(p.y, mm.y, vv.y, g.y, decay, w1, b2, w2, step_size, sbc2, eps);
      adamw_elem(p.z, mm.z, vv.z, g.z, decay, w1, b2, w2, step_size, sbc2, eps);
      adamw_elem(p.w, mm.w, vv.w, g.w, decay, w1, b2, w2, step_size, sbc2, eps);
      *reinterpret_cast<float4*>(master + f) = p;
      *reinterpret_cast<float4*>(m + f) = mm;
      *reinterpret_cast<float4*>(v + f) = vv;
      __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y), hi = __floats2bfloat162_rn(p.z, p.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(wp) = pk;
    } else {
      float p = master[f], mm = m[f], vv = v[f];
      adamw_elem(p, mm, vv, grad[f], decay, w1, b2, w2, step_size, sbc2, eps);
      master[f] = p;
      m[f] = mm;
      v[f] = vv;
      *wp = __float2bfloat16_rn(p);
    }
  }
}

// Scalar path (any segment layout)
__global__ void adamw_kernel(float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ grad, long long n, AdamSeg seg, float decay, float w1,
                             float b2, float w2, float step_size, float sbc2, float eps) {
  pdl_wait();
  pdl_trigger();
  __shared__ long long offs[65];
  for (int i = threadIdx.x; i <= seg.n_seg && i < 65; i += blockDim.x) offs[i] = seg.offsets[i];
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float p = master[i], mm = m[i], vv = v[i];
    adamw_elem(p, mm, vv, grad[i], decay, w1, b2, w2, step_size, sbc2, eps);
    master[i] = p;
    m[i] = mm;
    v[i] = vv;
    const int lo = seg_of(offs, seg.n_seg, i);
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

extern "C" int mace_dpo_scalar(mace_ctx* ctx, const double* delta_plus, const double* delta_minus, const double* beta,
                               int n, double* loss, double* margin, double* sig, void* stream) {
  if (n <= 0) return 0;
  if (!delta_plus || !delta_minus || !beta || !loss) return mace_fail(ctx, MACE_ERR_ARG, "dpo_scalar: null argument");
  launch_k(dpo_scalar_kernel, (n + 127) / 128, 128, 0, (cudaStream_t)stream, delta_plus, delta_minus, beta, n, loss, margin,
           sig);
  ctx->launches++;
  return mace_check_launch(ctx, "dpo_scalar");
}

extern "C" int mace_adamw_masked(mace_ctx* ctx, float* master, float* m, float* v, const float* grad, long long n,
                                 const long long* seg_offsets, void* const* seg_weights, int n_seg, float lr, float beta1,
                                 float beta2, float eps, float weight_decay, int step, void* stream) {
  return mace_adamw_masked2(ctx, master, m, v, grad, n, seg_offsets, seg_weights, n_seg, lr, beta1, beta2, eps,
                            weight_decay, step, 0, stream);
}

// hyper-parameters as doubles: the update's fp32 scalars are derived exactly as torch.optim.AdamW derives them
// from its Python floats (1 - lr*wd, 1 - beta1, 1 - beta2, lr / bc1, sqrt(bc2) in double, then rounded once)
extern "C" int mace_adamw_masked2(mace_ctx* ctx, float* master, float* m, float* v, const float* grad, long long n,
                                  const long long* seg_offsets, void* const* seg_weights, int n_seg, double lr,
                                  double beta1, double beta2, double eps, double weight_decay, int step, int vec4,
                                  void* stream) {
  if (n <= 0) return 0;
  if (n_seg > 64) return mace_fail(ctx, MACE_ERR_ARG, "adamw: at most 64 segments");
  if (step < 1) return mace_fail(ctx, MACE_ERR_ARG, "adamw: step is 1-based");
  const double bc1 = 1.0 - pow(beta1, step), bc2 = 1.0 - pow(beta2, step);
  AdamSeg seg{seg_offsets, reinterpret_cast<__nv_bfloat16* const*>(seg_weights), n_seg};
  const float decay = (float)(1.0 - lr * weight_decay), w1 = (float)(1.0 - beta1), b2 = (float)beta2,
              w2 = (float)(1.0 - beta2), ss = (float)(lr / bc1), sb = (float)sqrt(bc2), ep = (float)eps;
  const bool vec = vec4 && (n % 4 == 0) && ((uintptr_t)master % 16 == 0) && ((uintptr_t)m % 16 == 0) &&
                   ((uintptr_t)v % 16 == 0) && ((uintptr_t)grad % 16 == 0);
  if (vec) {  // caller asserts: every seg offset % 4 == 0 and every bf16 copy 8-byte aligned
    const long long n4 = n / 4;
    long long grid = (n4 + 511) / 512;
    if (grid > (long long)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    launch_k(adamw_vec_kernel, (int)grid, 256, 0, (cudaStream_t)stream, reinterpret_cast<float4*>(master),
             reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), reinterpret_cast<const float4*>(grad), n4, seg,
             decay, w1, b2, w2, ss, sb, ep);
  } else {
    int grid = (int)((n + 255) / 256);
    if (grid > ctx->num_sms * 8) grid = ctx->num_sms * 8;
    launch_k(adamw_kernel, grid, 256, 0, (cudaStream_t)stream, master, m, v, grad, n, seg, decay, w1, b2, w2, ss, sb, ep);
  }
  ctx->launches++;
  return mace_check_launch(ctx, "adamw");
}

extern "C" int mace_adamw_segments(mace_ctx* ctx, float* master, float* m, float* v, const float* grad, int n_seg,
                                   const long long* seg_vstart, const long long* seg_flat, void* const* seg_weights,
                                   long long n, double lr, double beta1, double beta2, double eps, double weight_decay,
                                   int step, int vec4, void* stream) {
  if (n <= 0 || n_seg <= 0) return 0;
  if (n_seg > 64) return mace_fail(ctx, MACE_ERR_ARG, "adamw_segments: at most 64 segments");
  if (step < 1) return mace_fail(ctx, MACE_ERR_ARG, "adamw_segments: step is 1-based");
  const double bc1 = 1.0 - pow(beta1, step), bc2 = 1.0 - pow(beta2, step);
  AdamSparse sg{seg_vstart, seg_flat, reinterpret_cast<__nv_bfloat16* const*>(seg_weights), n_seg};
  const float decay = (float)(1.0 - lr * weight_decay), w1 = (float)(1.0 - beta1), b2 = (float)beta2,
              w2 = (float)(1.0 - beta2), ss = (float)(lr / bc1), sb = (float)sqrt(bc2), ep = (float)eps;
  const bool vec = vec4 && n % 4 == 0;  // caller guarantees 4-aligned segments (offsets, lengths, bf16 copies)
  long long work = vec ? n / 4 : n;
  long long grid = (work + 255) / 256;
  if (grid > (long long)ctx->num_sms * 8) grid = ctx->num_sms * 8;
  if (vec)
    launch_k(adamw_sparse_kernel<true>, (int)grid, 256, 0, (cudaStream_t)stream, master, m, v, grad, n, sg, decay, w1, b2,
             w2, ss, sb, ep);
  else
    launch_k(adamw_sparse_kernel<false>, (int)grid, 256, 0, (cudaStream_t)stream, master, m, v, grad, n, sg, decay, w1, b2,
             w2, ss, sb, ep);
  ctx->launches++;
  return mace_check_launch(ctx, "adamw_segments");
}
