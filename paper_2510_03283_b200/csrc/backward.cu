// Backward kernels for the fine-tune rows of the hybrid batch: only FT rows, only
// the selected layers and above (the reference's "alignment-sensitive" update, PAPER.md:108-109 /
// alignment.py:168-172 stand-in). GEMM-shaped backward work (dX = dY.W, dW = dY^T.X) runs on the
// tcgen05 GEMM with MN-major operands; these are the row-wise and attention pieces.
//   norm_bwd    RMSNorm/LayerNorm: dx (+= into the residual grad, optional row scatter), dw/db partials
//   col_reduce  deterministic column sums of per-block partials (dw, db, bias grads)
//   act_bwd     SwiGLU / GELU(tanh)
//   rope_bwd    inverse rotation of dq/dk
//   attn_bwd    dense causal attention backward for FT sequences, head_dim 32 (head_dim 64 / 128: attention_bwd_tc.cu)
#include "common.cuh"
#include "mace_internal.h"

namespace mace {

// ------------------------------------------------------------------ norm backward
// rows i < n: x = xbuf[xrows ? xrows[i] : i], dy = dy[i]; dx written to dx[dxrows ? dxrows[i] : i] (+=).
// Per-block partials of dw (and db) go to part[blockIdx.x][0..d) and part[blockIdx.x][d..2d).
template <int kPerLane>
__global__ void __launch_bounds__(256, kPerLane <= 32 ? 2 : 1)
    norm_bwd_kernel(const float* __restrict__ x, int ldx, const int* __restrict__ xrows, const float* __restrict__ dy,
                    int lddy, int n, int d, const __nv_bfloat16* __restrict__ w, int layernorm, float eps,
                    float* __restrict__ dx, int lddx, const int* __restrict__ dxrows, float* __restrict__ part) {
  // one row per warp, 8 rows per CTA, float4 columns (lane owns columns 4 * (32 k + lane) .. + 3); the CTA's
  // dW / dB partials are merged in smem in warp order (deterministic) and reduced across CTAs by
  // col_reduce_kernel. No per-warp accumulator arrays: <= 128 registers at d 768, two CTAs per SM.
  constexpr int KV = kPerLane / 4;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31, nw = blockDim.x / 32;
  const int i = blockIdx.x * nw + warp;
  const bool active = i < n;
  // the norm weights do not depend on the previous kernel: fetched before the PDL wait (small d only;
  // at d 4096 the row alone fills the register file)
  constexpr bool kPre = KV <= 16;
  uint2 wraw[kPre ? KV : 1];
#pragma unroll
  for (int k = 0; k < (kPre ? KV : 0); ++k) {
    const int c = (k * 32 + lane) * 4;
    wraw[k] = active && c < d ? *reinterpret_cast<const uint2*>(w + c) : make_uint2(0u, 0u);
  }
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sh[];  // [2][d] block partials
  for (int c = threadIdx.x; c < 2 * d; c += blockDim.x) sh[c] = 0.f;
  float4 xv[KV], gv[KV];
  float rstd = 0.f;
  if (active) {
    const float* xr = x + (size_t)(xrows ? xrows[i] : i) * ldx;
    const float* gr = dy + (size_t)i * lddy;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int c = (k * 32 + lane) * 4;
      xv[k] = c < d ? *reinterpret_cast<const float4*>(xr + c) : z;
      gv[k] = c < d ? *reinterpret_cast<const float4*>(gr + c) : z;
      s += (xv[k].x + xv[k].y) + (xv[k].z + xv[k].w);
    }
    const float mean = layernorm ? warp_sum(s) / d : 0.f;
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int c = (k * 32 + lane) * 4;
      if (c < d) {
        xv[k].x -= mean; xv[k].y -= mean; xv[k].z -= mean; xv[k].w -= mean;
        ss += (xv[k].x * xv[k].x + xv[k].y * xv[k].y) + (xv[k].z * xv[k].z + xv[k].w * xv[k].w);
      }
    }
    rstd = rsqrtf(warp_sum(ss) / d + eps);
    auto gw_of = [&](int k, int c) {  // g * w of the lane's 4 columns
      const uint2 raw = kPre ? wraw[kPre ? k : 0] : *reinterpret_cast<const uint2*>(w + c);
      const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
      const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
      return make_float4(gv[k].x * w01.x, gv[k].y * w01.y, gv[k].z * w23.x, gv[k].w * w23.y);
    };
    float sum_g = 0.f, sum_gx = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int c = (k * 32 + lane) * 4;
      if (c < d) {
        const float4 gw = gw_of(k, c);
        sum_g += (gw.x + gw.y) + (gw.z + gw.w);
        sum_gx += (gw.x * xv[k].x * rstd + gw.y * xv[k].y * rstd) + (gw.z * xv[k].z * rstd + gw.w * xv[k].w * rstd);
      }
    }
    sum_g = warp_sum(sum_g) / d;
    sum_gx = warp_sum(sum_gx) / d;
    float* dr = dx + (size_t)(dxrows ? dxrows[i] : i) * lddx;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int c = (k * 32 + lane) * 4;
      if (c < d) {
        const float4 gw = gw_of(k, c);
        float4 o = *reinterpret_cast<float4*>(dr + c);
        const float h0 = xv[k].x * rstd, h1 = xv[k].y * rstd, h2 = xv[k].z * rstd, h3 = xv[k].w * rstd;
        if (layernorm) {
          o.x += rstd * (gw.x - sum_g - h0 * sum_gx);
          o.y += rstd * (gw.y - sum_g - h1 * sum_gx);
          o.z += rstd * (gw.z - sum_g - h2 * sum_gx);
          o.w += rstd * (gw.w - sum_g - h3 * sum_gx);
        } else {
          o.x += rstd * (gw.x - h0 * sum_gx);
          o.y += rstd * (gw.y - h1 * sum_gx);
          o.z += rstd * (gw.z - h2 * sum_gx);
          o.w += rstd * (gw.w - h3 * sum_gx);
        }
        *reinterpret_cast<float4*>(dr + c) = o;
      }
    }
  }
  __syncthreads();
  for (int wq = 0; wq < nw; ++wq) {
    if (warp == wq && active) {
#pragma unroll
      for (int k = 0; k < KV; ++k) {
        const int c = (k * 32 + lane) * 4;
        if (c < d) {
          sh[c] += gv[k].x * (xv[k].x * rstd);
          sh[c + 1] += gv[k].y * (xv[k].y * rstd);
          sh[c + 2] += gv[k].z * (xv[k].z * rstd);
          sh[c + 3] += gv[k].w * (xv[k].w * rstd);
          sh[d + c] += gv[k].x;
          sh[d + c + 1] += gv[k].y;
          sh[d + c + 2] += gv[k].z;
          sh[d + c + 3] += gv[k].w;
        }
      }
    }
    __syncthreads();
  }
  for (int c = threadIdx.x; c < 2 * d; c += blockDim.x) part[(size_t)blockIdx.x * 2 * d + c] = sh[c];
}

// out[c] += sum_b part[b * ld + c], deterministic: CTA = 32 columns x 8 row groups; group g sums partials
// b = g, g + 8, ... in order (4 independent chains), the 8 group sums are added in fixed order
__global__ void __launch_bounds__(256) col_reduce_kernel(const float* __restrict__ part, int nb, int ld, int ncols,
                                                         float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8][33];
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  if (c < ncols) {
    int k = 0;
    for (int b = g; b < nb; b += 8, ++k) s[k & 3] += part[(size_t)b * ld + c];
  }
  red[g][cl] = (s[0] + s[1]) + (s[2] + s[3]);
  __syncthreads();
  if (g == 0 && c < ncols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][cl];
    out[c] += t;
  }
}

// column sums of a bf16 matrix (bias grads), partial per row-chunk then col_reduce
__global__ void colsum_bf16_kernel(const __nv_bfloat16* __restrict__ y, int n, int N, int ld, int rows_per_block,
                                   float* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int r0 = blockIdx.y * rows_per_block, r1 = min(n, r0 + rows_per_block);
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 independent chains: loads in flight
  int r = r0;
  for (; r + 8 <= r1; r += 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] += __bfloat162float(y[(size_t)(r + i) * ld + c]);
  }
  for (int i = 0; r < r1; ++r, ++i) s[i] += __bfloat162float(y[(size_t)r * ld + c]);
  part[(size_t)blockIdx.y * N + c] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

// ------------------------------------------------------------------ activation backward
__global__ void act_bwd_kernel(const __nv_bfloat16* __restrict__ u, const __nv_bfloat16* __restrict__ da, int n, int F,
                               int swiglu, __nv_bfloat16* __restrict__ du) {
  pdl_wait();
  pdl_trigger();
  const size_t total = (size_t)n * F;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / F, c = i % F;
    const float g = __bfloat162float(da[i]);
    if (swiglu) {
      const float a = __bfloat162float(u[r * 2 * F + c]);
      const float b = __bfloat162float(u[r * 2 * F + F + c]);
      const float sg = 1.f / (1.f + __expf(-a));
      du[r * 2 * F + c] = __float2bfloat16(g * b * sg * (1.f + a * (1.f - sg)));
      du[r * 2 * F + F + c] = __float2bfloat16(g * a * sg);
    } else {
      const float x = __bfloat162float(u[i]);
      const float k0 = 0.7978845608028654f, k1 = 0.044715f;
      const float inner = k0 * (x + k1 * x * x * x);
      const float th = tanhf(inner);
      const float dgelu = 0.5f * (1.f + th) + 0.5f * x * (1.f - th * th) * k0 * (1.f + 3.f * k1 * x * x);
      du[i] = __float2bfloat16(g * dgelu);
    }
  }
}

// ------------------------------------------------------------------ RoPE backward on dq / dk (fp32 rows)
__global__ void rope_bwd_kernel(float* __restrict__ dqkv, int n, int Hq, int Hkv, int hd, const int* __restrict__ pos,
                                const float* __restrict__ cos_t, const float* __restrict__ sin_t) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (r >= n) return;
  const int W = (Hq + 2 * Hkv) * hd, half = hd / 2;
  float* row = dqkv + (size_t)r * W;
  const int p = pos[r];
  for (int idx = threadIdx.x; idx < (Hq + Hkv) * half; idx += blockDim.x) {
    const int h = idx / half, i = idx % half;
    float* b = row + h * hd;
    const float c = cos_t[(size_t)p * half + i], s = sin_t[(size_t)p * half + i];
    const float g1 = b[i], g2 = b[i + half];
    b[i] = g1 * c + g2 * s;
    b[i + half] = -g1 * s + g2 * c;
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, long long n, __nv_bfloat16* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16(x[i]);
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ x, long long n, float* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = __bfloat162float(x[i]);
}

// ------------------------------------------------------------------ attention backward (dense FT sequences)
// D[r, hq] = sum_d dO[r, hq, d] * O[r, hq, d]
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout, int n,
                                     int Hq, int hd, float* __restrict__ Dout) {
  pdl_wait();
  pdl_trigger();
  const int idx = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (idx >= n * Hq) return;
  const __nv_bfloat16* a = o + (size_t)idx * hd;
  const __nv_bfloat16* b = dout + (size_t)idx * hd;
  float s = 0.f;
  for (int c = lane; c < hd; c += 32) s += __bfloat162float(a[c]) * __bfloat162float(b[c]);
  s = warp_sum(s);
  if (lane == 0) Dout[idx] = s;
}

// block = (seq, kv head h, key block jb of 64). Loops over the G query heads of the group and the
// query chunks at or after the key block (causal). K/V block fp32 in smem.
template <int HD>
__global__ void __launch_bounds__(256) attn_bwd_kernel(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
                                                       const float* __restrict__ lse, const float* __restrict__ Dv,
                                                       const MaceSeq* __restrict__ seqs, const int4* __restrict__ items,
                                                       int Hq, int Hkv, float scale, float* __restrict__ dqkv,
                                                       int row_offset, int* __restrict__ dq_order) {
  pdl_wait();
  pdl_trigger();
  constexpr int B = 64;
  constexpr int LDH = HD + 1;
  extern __shared__ float sm[];
  float* Ks = sm;                 // [B][LDH]
  float* Vs = Ks + B * LDH;       // [B][LDH]
  float* Qs = Vs + B * LDH;       // [B][LDH]
  float* dOs = Qs + B * LDH;      // [B][LDH]
  float* Ps = dOs + B * LDH;      // [B][B+1]  P[q][k]
  float* dSs = Ps + B * (B + 1);  // [B][B+1]
  float* ls = dSs + B * (B + 1);  // [B] lse
  float* Ds = ls + B;             // [B]

  const int4 it = items[blockIdx.x];
  const MaceSeq sq = seqs[it.x];
  const int h = it.y, jb = it.z;
  const int G = Hq / Hkv;
  const int W = (Hq + 2 * Hkv) * HD;
  const int n = sq.q_len;
  const int base = sq.q_start - row_offset;  // local row of token 0 in the FT activation block
  const int h1 = sq.hole_len > 0 ? sq.hole0 + sq.hole_len : n + 1;  // preference-pair hole (MaceSeq)
  const int k0 = jb * B;
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;  // 16x16 threads, 4x4 micro tiles

  for (int i = tid; i < B * HD; i += 256) {
    const int r = i / HD, c = i % HD;
    const bool ok = k0 + r < n;
    const __nv_bfloat16* row = qkv + (size_t)(base + k0 + r) * W;
    Ks[r * LDH + c] = ok ? __bfloat162float(row[(Hq + h) * HD + c]) : 0.f;
    Vs[r * LDH + c] = ok ? __bfloat162float(row[(Hq + Hkv + h) * HD + c]) : 0.f;
  }
  // dK / dV accumulators: thread owns key rows ty*4..+3, dims tx*(HD/16)..
  constexpr int DC = HD / 16;
  float dK[4][DC], dV[4][DC];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < DC; ++b) dK[a][b] = dV[a][b] = 0.f;

  // query chunks at or after the key block, LAST chunk first (outer), the GQA group's heads inner: every key block
  // reaches a given (query chunk, head) at the same iteration, so the ordered dQ hand-off does not accumulate lag
  const int q_last = (n - 1) / B * B;
  for (int q0 = q_last; q0 >= k0; q0 -= B)
  for (int g = 0; g < G; ++g) {
    const int hq = h * G + g;
    {
      __syncthreads();
      for (int i = tid; i < B * HD; i += 256) {
        const int r = i / HD, c = i % HD;
        const bool ok = q0 + r < n;
        Qs[r * LDH + c] = ok ? __bfloat162float(qkv[(size_t)(base + q0 + r) * W + hq * HD + c]) : 0.f;
        dOs[r * LDH + c] = ok ? __bfloat162float(dout[(size_t)(base + q0 + r) * Hq * HD + hq * HD + c]) : 0.f;
      }
      for (int i = tid; i < B; i += 256) {
        const bool ok = q0 + i < n;
        ls[i] = ok ? lse[(size_t)(base + q0 + i) * Hq + hq] : 0.f;
        Ds[i] = ok ? Dv[(size_t)(base + q0 + i) * Hq + hq] : 0.f;
      }
      __syncthreads();
      // S = Q K^T, dP = dO V^T : thread computes q rows ty*4.., key cols tx*4..
      float s[4][4], dp[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) s[a][b] = dp[a][b] = 0.f;
      for (int d = 0; d < HD; ++d) {
        float qa[4], ka[4], oa[4], va[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          qa[a] = Qs[(ty * 4 + a) * LDH + d];
          oa[a] = dOs[(ty * 4 + a) * LDH + d];
          ka[a] = Ks[(tx * 4 + a) * LDH + d];
          va[a] = Vs[(tx * 4 + a) * LDH + d];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            s[a][b] = fmaf(qa[a], ka[b], s[a][b]);
            dp[a][b] = fmaf(oa[a], va[b], dp[a][b]);
          }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int qi = ty * 4 + a, qg = q0 + qi;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int kj = tx * 4 + b, kg = k0 + kj;
          float p = 0.f;
          if (qg < n && kg < n && kg <= qg && !(qg >= h1 && kg >= sq.hole0 && kg < h1))
            p = __expf(s[a][b] * scale - ls[qi]);
          Ps[qi * (B + 1) + kj] = p;
          dSs[qi * (B + 1) + kj] = p * (dp[a][b] - Ds[qi]);
        }
      }
      __syncthreads();
      // dV += P^T dO ; dK += dS^T Q * scale   (thread: key rows ty*4.., dims tx*DC..)
      for (int qi = 0; qi < B; ++qi) {
        float pa[4], sa[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          pa[a] = Ps[qi * (B + 1) + ty * 4 + a];
          sa[a] = dSs[qi * (B + 1) + ty * 4 + a];
        }
#pragma unroll
        for (int b = 0; b < DC; ++b) {
          const float o_ = dOs[qi * LDH + tx * DC + b];
          const float q_ = Qs[qi * LDH + tx * DC + b];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            dV[a][b] = fmaf(pa[a], o_, dV[a][b]);
            dK[a][b] = fmaf(sa[a], q_, dK[a][b]);
          }
        }
      }
      // dQ += dS K * scale  (thread: q rows ty*4.., dims tx*DC..) -> atomics (G x key blocks contribute)
      float dq[4][DC];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < DC; ++b) dq[a][b] = 0.f;
      for (int kj = 0; kj < B; ++kj) {
        float sa[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) sa[a] = dSs[(ty * 4 + a) * (B + 1) + kj];
#pragma unroll
        for (int b = 0; b < DC; ++b) {
          const float k_ = Ks[kj * LDH + tx * DC + b];
#pragma unroll
          for (int a = 0; a < 4; ++a) dq[a][b] = fmaf(sa[a], k_, dq[a][b]);
        }
      }
      // key blocks jb = 0..q0/B contribute to this query chunk: with dq_order in ascending jb (bitwise reproducible)
      int* ctr = dq_order ? dq_order + (size_t)(base + q0) * Hq + hq : nullptr;
      if (ctr) {
        if (tid == 0) order_wait(ctr, jb);
        __syncthreads();
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int qg = q0 + ty * 4 + a;
        if (qg < n) {
#pragma unroll
          for (int b = 0; b < DC; ++b) {
            float* p = &dqkv[(size_t)(base + qg) * W + hq * HD + tx * DC + b];
            if (ctr)
              __stcg(p, __ldcg(p) + dq[a][b] * scale);
            else
              atomicAdd(p, dq[a][b] * scale);
          }
        }
      }
      if (ctr) {
        __threadfence();
        __syncthreads();
        if (tid == 0) order_release(ctr, jb == q0 / B ? 0 : jb + 1);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int kg = k0 + ty * 4 + a;
    if (kg < n) {
#pragma unroll
      for (int b = 0; b < DC; ++b) {
        dqkv[(size_t)(base + kg) * W + (Hq + h) * HD + tx * DC + b] = dK[a][b] * scale;
        dqkv[(size_t)(base + kg) * W + (Hq + Hkv + h) * HD + tx * DC + b] = dV[a][b];
      }
    }
  }
}

}  // namespace mace

using namespace mace;

extern "C" int mace_norm_bwd(mace_ctx* ctx, const float* x, int ldx, const int* xrows, const float* dy, int lddy, int n,
                             int d, const void* w, int layernorm, float eps, float* dx, int lddx, const int* dxrows,
                             float* dw, float* db, float* workspace, size_t workspace_bytes, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int rows_per_block = 8;  // one row per warp: n/8 CTAs keep every SM busy
  const int nb = (n + rows_per_block - 1) / rows_per_block;
  if (workspace_bytes < (size_t)nb * 2 * d * 4) return mace_fail(ctx, MACE_ERR_ARG, "norm_bwd: workspace too small");
  if ((d | ldx | lddy | lddx) & 3) return mace_fail(ctx, MACE_ERR_ARG, "norm_bwd: d and leading dims must be multiples of 4");
  const int per_lane = (d + 127) / 128 * 4;  // float4 columns per lane, times 4
  const size_t sh = 2 * d * sizeof(float);
  auto* W = (const __nv_bfloat16*)w;
#define MACE_NB(K) launch_k(norm_bwd_kernel<K>, nb, 256, sh, s, x, ldx, xrows, dy, lddy, n, d, W, layernorm, eps, dx, lddx, dxrows, workspace)
  if (per_lane <= 8) MACE_NB(8);
  else if (per_lane <= 24) MACE_NB(24);
  else if (per_lane <= 64) MACE_NB(64);
  else if (per_lane <= 128) MACE_NB(128);
  else return mace_fail(ctx, MACE_ERR_ARG, "norm_bwd: d too large");
#undef MACE_NB
  ctx->launches++;
  if (dw) {  // NULL: frozen norm (LoRA mode trains only the adapters)
    launch_k(col_reduce_kernel, (d + 31) / 32, 256, 0, s, workspace, nb, 2 * d, d, dw);
    ctx->launches++;
  }
  if (layernorm && db) {
    launch_k(col_reduce_kernel, (d + 31) / 32, 256, 0, s, workspace + d, nb, 2 * d, d, db);
    ctx->launches++;
  }
  return mace_check_launch(ctx, "norm_bwd");
}

extern "C" int mace_colsum_bf16(mace_ctx* ctx, const void* y, int n, int N, int ld, float* out, float* workspace,
                                size_t workspace_bytes, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int rpb = 64;
  const int nb = (n + rpb - 1) / rpb;
  if (workspace_bytes < (size_t)nb * N * 4) return mace_fail(ctx, MACE_ERR_ARG, "colsum: workspace too small");
  launch_k(colsum_bf16_kernel, dim3((N + 255) / 256, nb), 256, 0, s, (const __nv_bfloat16*)y, n, N, ld, rpb, workspace);
  launch_k(col_reduce_kernel, (N + 31) / 32, 256, 0, s, workspace, nb, N, N, out);
  ctx->launches += 2;
  return mace_check_launch(ctx, "colsum");
}

extern "C" int mace_act_bwd(mace_ctx* ctx, const void* u, const void* da, int n, int F, int swiglu, void* du,
                            void* stream) {
  if (n <= 0) return 0;
  int grid = (int)(((size_t)n * F + 255) / 256);
  if (grid > ctx->num_sms * 16) grid = ctx->num_sms * 16;
  launch_k(act_bwd_kernel, grid, 256, 0, (cudaStream_t)stream, (const __nv_bfloat16*)u, (const __nv_bfloat16*)da, n, F, swiglu,
                                                         (__nv_bfloat16*)du);
  ctx->launches++;
  return mace_check_launch(ctx, "act_bwd");
}

extern "C" int mace_rope_bwd(mace_ctx* ctx, float* dqkv, int n, int Hq, int Hkv, int hd, const int* pos,
                             const float* cos_t, const float* sin_t, void* stream) {
  if (n <= 0) return 0;
  launch_k(rope_bwd_kernel, n, 128, 0, (cudaStream_t)stream, dqkv, n, Hq, Hkv, hd, pos, cos_t, sin_t);
  ctx->launches++;
  return mace_check_launch(ctx, "rope_bwd");
}

extern "C" int mace_f32_to_bf16(mace_ctx* ctx, const float* x, long long n, void* y, void* stream) {
  if (n <= 0) return 0;
  long long grid = (n + 255) / 256;
  if (grid > ctx->num_sms * 16) grid = ctx->num_sms * 16;
  launch_k(f32_to_bf16_kernel, (int)grid, 256, 0, (cudaStream_t)stream, x, n, (__nv_bfloat16*)y);
  ctx->launches++;
  return mace_check_launch(ctx, "f32_to_bf16");
}

extern "C" int mace_bf16_to_f32(mace_ctx* ctx, const void* x, long long n, float* y, void* stream) {
  if (n <= 0) return 0;
  long long grid = (n + 255) / 256;
  if (grid > ctx->num_sms * 16) grid = ctx->num_sms * 16;
  launch_k(bf16_to_f32_kernel, (int)grid, 256, 0, (cudaStream_t)stream, (const __nv_bfloat16*)x, n, y);
  ctx->launches++;
  return mace_check_launch(ctx, "bf16_to_f32");
}

namespace mace {
int attn_bwd_tc(MaceCtx* ctx, const void* qkv, const void* dout, const float* lse, int n_rows, int Hq, int Hkv, int hd,
                const MaceSeq* seqs, const int* items, int n_items, int row_offset, const float* Dbuf, float* dqkv,
                int* dq_order, cudaStream_t s);  // attention_bwd_tc.cu
}  // namespace mace

// items int4 [n_items] = (seq, kv_head, key_block, steps); key blocks of 128 keys (head_dim 64 / 128: the tcgen05
// kernel of attention_bwd_tc.cu) or 64 keys (head_dim 32: the CUDA-core kernel below). Rows of qkv/dout/lse/dqkv
// are local to the FT
// block starting at global row `row_offset`. dqkv must be zeroed by the caller (dq accumulates).
extern "C" int mace_attn_bwd2(mace_ctx* ctx, const void* qkv, const void* o, const void* dout, const float* lse,
                              int n_rows, int Hq, int Hkv, int hd, const MaceSeq* seqs, const int* items, int n_items,
                              int row_offset, float* Dbuf, float* dqkv, int* dq_order, void* stream) {
  if (n_items <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  launch_k(attn_bwd_prep_kernel, (n_rows * Hq + 7) / 8, 256, 0, s, (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, n_rows,
                                                             Hq, hd, Dbuf);
  if (hd == 64 || hd == 128) {  // tcgen05 path (128-key blocks)
    const int rc = attn_bwd_tc(ctx, qkv, dout, lse, n_rows, Hq, Hkv, hd, seqs, items, n_items, row_offset, Dbuf, dqkv,
                               dq_order, s);
    if (rc) return rc;
    ctx->launches++;  // the prep kernel
    return mace_check_launch(ctx, "attn_bwd");
  }
  const float scale = 1.f / sqrtf((float)hd);
  auto go = [&](auto kern, int HD) {
    const size_t sh = (4 * 64 * (HD + 1) + 2 * 64 * 65 + 128) * sizeof(float);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
    launch_k(kern, n_items, 256, sh, s, (const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dout, lse, Dbuf, seqs,
                                  reinterpret_cast<const int4*>(items), Hq, Hkv, scale, dqkv, row_offset, dq_order);
  };
  switch (hd) {
    case 32: go(attn_bwd_kernel<32>, 32); break;
    case 64: go(attn_bwd_kernel<64>, 64); break;
    case 128: go(attn_bwd_kernel<128>, 128); break;
    default: return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn_bwd: head_dim");
  }
  ctx->launches += 2;
  return mace_check_launch(ctx, "attn_bwd");
}

extern "C" int mace_attn_bwd(mace_ctx* ctx, const void* qkv, const void* o, const void* dout, const float* lse, int n_rows,
                             int Hq, int Hkv, int hd, const MaceSeq* seqs, const int* items, int n_items, int row_offset,
                             float* Dbuf, float* dqkv, void* stream) {
  return mace_attn_bwd2(ctx, qkv, o, dout, lse, n_rows, Hq, Hkv, hd, seqs, items, n_items, row_offset, Dbuf, dqkv,
                        nullptr, stream);
}
