// Row-wise fused kernels of the hybrid step (HBM-bound; one warp per row, 16-byte vector access).
//   embed          tokens -> fp32 residual stream (+ learned positions for GPT-2)
//   norm           fp32 residual -> bf16 RMSNorm/LayerNorm output, optional row gather
//   rope_kv        RoPE on q/k (Llama) in the packed qkv rows + scatter of k/v rows into the
//                  head-major paged KV pools (prefill rows -> prompt pages, decode rows -> the
//                  per-head decode ring), replacing the MB bookkeeping of engine.py:469-471,512-514
//   act            SwiGLU / GELU(tanh)
//   argmax         greedy token per decode row (ties -> lowest id, = torch.argmax)
#include "common.cuh"
#include "mace_internal.h"

namespace mace {

// ------------------------------------------------------------------ embed
// tokens[row] < 0 means "the token this request's slot produced last tick": last_token[-tok-1]
// (decode input feedback stays on the device; no host round trip per tick)
__global__ void embed_kernel(const int* __restrict__ tokens, const int* __restrict__ pos,
                             const int* __restrict__ last_token, const __nv_bfloat16* __restrict__ emb,
                             const __nv_bfloat16* __restrict__ pos_emb, int T, int d, float* __restrict__ x) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (row >= T) return;
  const int lane = threadIdx.x & 31;
  int tok = tokens[row];
  if (tok < 0) tok = last_token[-tok - 1];
  const __nv_bfloat16* e = emb + (size_t)tok * d;
  const __nv_bfloat16* pe = pos_emb ? pos_emb + (size_t)pos[row] * d : nullptr;
  float* xr = x + (size_t)row * d;
  for (int c = lane * 8; c < d; c += 256) {
    uint4 u = *reinterpret_cast<const uint4*>(e + c);
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(h[j]);
    if (pe) {
      uint4 up = *reinterpret_cast<const uint4*>(pe + c);
      const __nv_bfloat16* hp = reinterpret_cast<const __nv_bfloat16*>(&up);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += __bfloat162float(hp[j]);
    }
    *reinterpret_cast<float4*>(xr + c) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(xr + c + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// ------------------------------------------------------------------ norm, wide rows (d >= 2048)
// One 256-thread CTA per row: thread t owns columns 4 (t + 256 j), j < kVec (d = 1024 kVec) -- a few float4 of the
// row in registers (the warp-per-row kernel below would hold d / 32 floats per lane: 128 at d 4096, which
// spills or starves occupancy). Statistics through a two-level (warp, then CTA) reduction in fixed order.
template <int kVec>
__global__ void __launch_bounds__(256) norm_wide_kernel(const float* __restrict__ x, int ldx, const int* __restrict__ rows,
                                                        int n_rows, int d, const __nv_bfloat16* __restrict__ w,
                                                        const __nv_bfloat16* __restrict__ b, int layernorm, float eps,
                                                        __nv_bfloat16* __restrict__ out, int ldo,
                                                        float* __restrict__ rstd_out) {
  __shared__ float red[2][8];
  const int i = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint2 wr[kVec], br[kVec];
#pragma unroll
  for (int j = 0; j < kVec; ++j) {  // weights: independent of the previous kernel, fetched before the PDL wait
    const int c = 4 * (t + 256 * j);
    wr[j] = *reinterpret_cast<const uint2*>(w + c);
    br[j] = layernorm ? *reinterpret_cast<const uint2*>(b + c) : make_uint2(0u, 0u);
  }
  pdl_wait();
  pdl_trigger();
  const float* xr = x + (size_t)(rows ? rows[i] : i) * ldx;
  float4 v[kVec];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    v[j] = *reinterpret_cast<const float4*>(xr + 4 * (t + 256 * j));
    s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
  }
  float mean = 0.f;
  if (layernorm) {
    s = warp_sum(s);
    if (lane == 0) red[0][warp] = s;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) tot += red[0][k];
    mean = tot / d;
  }
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const float a = v[j].x - mean, bq = v[j].y - mean, c = v[j].z - mean, e = v[j].w - mean;
    ss += (a * a + bq * bq) + (c * c + e * e);
  }
  ss = warp_sum(ss);
  if (lane == 0) red[1][warp] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) tot += red[1][k];
  const float rstd = rsqrtf(tot / d + eps);
  if (rstd_out && t == 0) rstd_out[i] = rstd;
  __nv_bfloat16* o = out + (size_t)i * ldo;
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const __nv_bfloat16* wk = reinterpret_cast<const __nv_bfloat16*>(&wr[j]);
    const __nv_bfloat16* bk = reinterpret_cast<const __nv_bfloat16*>(&br[j]);
    const float f[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
    float y[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      y[q] = (f[q] - mean) * rstd * __bfloat162float(wk[q]);
      if (layernorm) y[q] += __bfloat162float(bk[q]);
    }
    *reinterpret_cast<uint2*>(o + 4 * (t + 256 * j)) = make_uint2(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]));
  }
}

// ------------------------------------------------------------------ norm (fp32 in -> bf16 out)
// out[i] = norm(x[rows ? rows[i] : i]); LayerNorm when bias != nullptr semantics chosen by `layernorm`.
template <int kPerLane>
__global__ void norm_kernel(const float* __restrict__ x, int ldx, const int* __restrict__ rows, int n_rows, int d,
                            const __nv_bfloat16* __restrict__ w, const __nv_bfloat16* __restrict__ b, int layernorm,
                            float eps, __nv_bfloat16* __restrict__ out, int ldo, float* __restrict__ rstd_out) {
  const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  // the weights do not depend on the previous kernel: fetched before the PDL wait, under its tail
  // (up to d 2048; at d 4096 they are read after the statistics, keeping the row in registers)
  constexpr int KV = kPerLane / 4;
  constexpr bool kPre = KV <= 16;
  uint2 wr[KV], br[KV];
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int c = (k * 32 + lane) * 4;
    wr[k] = br[k] = make_uint2(0u, 0u);
    if (kPre && c < d && i < n_rows) {
      wr[k] = *reinterpret_cast<const uint2*>(w + c);
      if (layernorm) br[k] = *reinterpret_cast<const uint2*>(b + c);
    }
  }
  pdl_wait();
  pdl_trigger();
  if (i >= n_rows) return;
  const int src = rows ? rows[i] : i;
  const float* xr = x + (size_t)src * ldx;
  float v[kPerLane];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kPerLane / 4; ++k) {
    const int c = (k * 32 + lane) * 4;
    float4 f = c < d ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    v[4 * k] = f.x; v[4 * k + 1] = f.y; v[4 * k + 2] = f.z; v[4 * k + 3] = f.w;
    s += f.x + f.y + f.z + f.w;
  }
  float mean = 0.f;
  if (layernorm) {
    mean = warp_sum(s) / d;
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kPerLane / 4; ++k) {
    const int c = (k * 32 + lane) * 4;
    if (c < d) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float t = v[4 * k + j] - mean;
        ss += t * t;
      }
    }
  }
  const float rstd = rsqrtf(warp_sum(ss) / d + eps);
  if (rstd_out && lane == 0) rstd_out[i] = rstd;
  __nv_bfloat16* o = out + (size_t)i * ldo;
#pragma unroll
  for (int k = 0; k < kPerLane / 4; ++k) {
    const int c = (k * 32 + lane) * 4;
    if (c < d) {
      if (!kPre) {
        wr[k] = *reinterpret_cast<const uint2*>(w + c);
        if (layernorm) br[k] = *reinterpret_cast<const uint2*>(b + c);
      }
      const __nv_bfloat16* wk = reinterpret_cast<const __nv_bfloat16*>(&wr[k]);
      const __nv_bfloat16* bk = reinterpret_cast<const __nv_bfloat16*>(&br[k]);
      float y[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        y[j] = (v[4 * k + j] - mean) * rstd * __bfloat162float(wk[j]);
        if (layernorm) y[j] += __bfloat162float(bk[j]);
      }
      uint2 pk = make_uint2(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]));
      *reinterpret_cast<uint2*>(o + c) = pk;
    }
  }
}

// ------------------------------------------------------------------ RoPE + paged KV write
// qkv row layout: [q heads | k heads | v heads] x hd (bf16). cos/sin tables [n_pos, hd/2] fp32.
// Row kinds come from the tick's sequence table (MaceSeq). Paged destinations:
//   prefill row (kind 0), prompt index t: head page = ptab[slot][t/16] * Hkv + h, row t % 16
//   decode row  (kind 1), decode slot j:  head page = dtab[slot][h][(j - dec_base)/16],  row (j - dec_base) % 16
//   fine-tune row (kind 2): attention reads K/V straight from the qkv rows (no write)
// One CTA per row; every memory access is 16 bytes. Work items of a row:
//   rotation items (q and k heads; only with RoPE): 8 consecutive pairs (i, i + hd/2) of one head -- two uint4
//     loads, two float4 pairs of cos / sin, two uint4 stores back into the row; a k item also stores both rotated
//     chunks straight into its KV page (no re-read of the row)
//   copy items: the v heads' 16-byte chunks (and, without RoPE, the k heads' too) -> KV pages
__device__ __forceinline__ long long kv_page_row(const MaceSeq& sq, const MaceKvLayout& kv, int Hkv, int h, int t,
                                                 int hd) {
  int page, row;
  if (sq.kind == 0) {
    page = kv.ptab[(size_t)sq.slot * kv.max_prompt_pages + t / kPageTokens] * Hkv + h;
    row = t % kPageTokens;
  } else {  // ring offset relative to dec_base (any value after a compaction re-base, mace_kv_compact)
    const int rel = t - kv.dec_base[sq.slot * Hkv + h];
    page = kv.dtab[((size_t)sq.slot * Hkv + h) * kv.max_dec_pages + rel / kPageTokens];
    row = rel % kPageTokens;
  }
  return ((long long)page * kPageTokens + row) * hd;
}

__global__ void __launch_bounds__(128) rope_kv_kernel(__nv_bfloat16* __restrict__ qkv, int T, int Hq, int Hkv, int hd,
                                                      const int* __restrict__ row_pos, const int* __restrict__ row_seq,
                                                      const int* __restrict__ row_kvi, const MaceSeq* __restrict__ seqs,
                                                      const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                                      int apply_rope, const MaceKvLayout kv,
                                                      __nv_bfloat16* __restrict__ k_pool,
                                                      __nv_bfloat16* __restrict__ v_pool) {
  const int row = blockIdx.x;
  // row metadata and page tables are written before the tick's first layer: read under the PDL overlap
  const MaceSeq sq = seqs[row_seq[row]];
  const bool paged = sq.kind != 2 && k_pool != nullptr;
  const int t = paged ? row_kvi[row] : 0;
  const int pos = row_pos[row];
  pdl_wait();
  pdl_trigger();
  const int half = hd / 2, cph = half / 8;  // rotation chunks per head
  __nv_bfloat16* r = qkv + (size_t)row * (Hq + 2 * Hkv) * hd;
  const int n_rot = apply_rope ? (Hq + Hkv) * cph : 0;
  const int n_copy = paged ? (apply_rope ? Hkv : 2 * Hkv) * (hd / 8) : 0;
  for (int it = threadIdx.x; it < n_rot + n_copy; it += blockDim.x) {
    if (it < n_rot) {
      const int h = it / cph, i0 = (it % cph) * 8;
      __nv_bfloat16* base = r + h * hd;
      uint4 a = *reinterpret_cast<const uint4*>(base + i0);
      uint4 b = *reinterpret_cast<const uint4*>(base + half + i0);
      const float4* cp = reinterpret_cast<const float4*>(cos_t + (size_t)pos * half + i0);
      const float4* sp = reinterpret_cast<const float4*>(sin_t + (size_t)pos * half + i0);
      const float4 c0 = cp[0], c1 = cp[1], s0 = sp[0], s1 = sp[1];
      const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
      const __nv_bfloat16* ah = reinterpret_cast<const __nv_bfloat16*>(&a);
      const __nv_bfloat16* bh = reinterpret_cast<const __nv_bfloat16*>(&b);
      float o1[8], o2[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float x1 = __bfloat162float(ah[j]), x2 = __bfloat162float(bh[j]);
        o1[j] = x1 * cs[j] - x2 * sn[j];
        o2[j] = x2 * cs[j] + x1 * sn[j];
      }
      const uint4 p1 = make_uint4(pack_bf16(o1[0], o1[1]), pack_bf16(o1[2], o1[3]), pack_bf16(o1[4], o1[5]),
                                  pack_bf16(o1[6], o1[7]));
      const uint4 p2 = make_uint4(pack_bf16(o2[0], o2[1]), pack_bf16(o2[2], o2[3]), pack_bf16(o2[4], o2[5]),
                                  pack_bf16(o2[6], o2[7]));
      *reinterpret_cast<uint4*>(base + i0) = p1;
      *reinterpret_cast<uint4*>(base + half + i0) = p2;
      if (paged && h >= Hq) {  // a k head: the rotated chunks go to its page as well
        const long long dst = kv_page_row(sq, kv, Hkv, h - Hq, t, hd);
        *reinterpret_cast<uint4*>(k_pool + dst + i0) = p1;
        *reinterpret_cast<uint4*>(k_pool + dst + half + i0) = p2;
      }
    } else {
      const int c = it - n_rot, per = hd / 8;
      // with RoPE only v heads are copied; without it k heads first, then v heads
      const int hh = c / per, e = (c % per) * 8;
      const bool is_v = apply_rope || hh >= Hkv;
      const int h = apply_rope ? hh : (hh % Hkv);
      const long long dst = kv_page_row(sq, kv, Hkv, h, t, hd);
      const uint4 u = *reinterpret_cast<const uint4*>(r + (Hq + (is_v ? Hkv : 0) + h) * hd + e);
      *reinterpret_cast<uint4*>((is_v ? v_pool : k_pool) + dst + e) = u;
    }
  }
}

// ------------------------------------------------------------------ activations
// llama: up row = [gate(F) | up(F)] -> silu(gate) * up ; gpt2: gelu_tanh(up)
__global__ void act_kernel(const __nv_bfloat16* __restrict__ u, int T, int F, int swiglu,
                           __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const size_t total = (size_t)T * F / 8;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t row = (i * 8) / F, c = (i * 8) % F;
    const int W = swiglu ? 2 * F : F;
    uint4 a = *reinterpret_cast<const uint4*>(u + row * W + c);
    const __nv_bfloat16* ah = reinterpret_cast<const __nv_bfloat16*>(&a);
    float y[8];
    if (swiglu) {
      uint4 b = *reinterpret_cast<const uint4*>(u + row * W + F + c);
      const __nv_bfloat16* bh = reinterpret_cast<const __nv_bfloat16*>(&b);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float g = __bfloat162float(ah[j]);
        y[j] = g / (1.f + __expf(-g)) * __bfloat162float(bh[j]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float x = __bfloat162float(ah[j]);
        y[j] = 0.5f * x * (1.f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
      }
    }
    *reinterpret_cast<uint4*>(out + row * F + c) =
        make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]), pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7]));
  }
}

// ------------------------------------------------------------------ keys of the fused lm_head argmax -> token ids
__global__ void argmax_keys_kernel(unsigned long long* __restrict__ keys, int n, int* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    out[i] = (int)(0xffffffffu - (uint32_t)(keys[i] & 0xffffffffull));
    keys[i] = 0ull;  // ready for the next MACE_EPI_ARGMAX GEMM
  }
}

// ------------------------------------------------------------------ argmax over fp32 logits rows
__global__ void argmax_kernel(const float* __restrict__ logits, int V, int ld, int* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const float* r = logits + (size_t)blockIdx.x * ld;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int c = threadIdx.x; c < V; c += blockDim.x) {
    const float v = r[c];
    if (v > best) {
      best = v;
      idx = c;
    }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) {
      best = ob;
      idx = oi;
    }
  }
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) {
    sb[w] = best;
    si[w] = idx;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x / 32;
    best = (threadIdx.x < nw) ? sb[threadIdx.x] : -INFINITY;
    idx = (threadIdx.x < nw) ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ob > best || (ob == best && oi < idx)) {
        best = ob;
        idx = oi;
      }
    }
    if (threadIdx.x == 0) out[blockIdx.x] = idx;
  }
}

}  // namespace mace

using namespace mace;

extern "C" int mace_embed(mace_ctx* ctx, const int* tokens, const int* pos, const int* last_token, const void* emb,
                          const void* pos_emb, int T, int d, float* x, void* stream) {
  if (T <= 0) return 0;
  if (d % 256) return mace_fail(ctx, MACE_ERR_ARG, "embed: d must be a multiple of 256");
  launch_k(embed_kernel, (T + 7) / 8, 256, 0, (cudaStream_t)stream, tokens, pos, last_token, (const __nv_bfloat16*)emb,
                                                                 (const __nv_bfloat16*)pos_emb, T, d, x);
  ctx->launches++;
  return mace_check_launch(ctx, "embed");
}

extern "C" int mace_norm(mace_ctx* ctx, const float* x, int ldx, const int* rows, int n_rows, int d, const void* w,
                         const void* b, int layernorm, float eps, void* out, int ldo, float* rstd_out, void* stream) {
  if (n_rows <= 0) return 0;
  if (d % 128) return mace_fail(ctx, MACE_ERR_ARG, "norm: d must be a multiple of 128");
  const int per_lane = (d + 31) / 32;
  dim3 grid((n_rows + 7) / 8);
  auto* W = (const __nv_bfloat16*)w;
  auto* B = (const __nv_bfloat16*)b;
  auto* O = (__nv_bfloat16*)out;
  cudaStream_t s = (cudaStream_t)stream;
  if (d % 1024 == 0 && d >= 2048 && d <= 8192 && (ldx % 4) == 0 && (ldo % 4) == 0) {
#define MACE_NW(K) launch_k(norm_wide_kernel<K>, dim3(n_rows), 256, 0, s, x, ldx, rows, n_rows, d, W, B, layernorm, eps, O, ldo, rstd_out)
    switch (d / 1024) {
      case 2: MACE_NW(2); break;
      case 3: MACE_NW(3); break;
      case 4: MACE_NW(4); break;
      case 5: MACE_NW(5); break;
      case 6: MACE_NW(6); break;
      case 7: MACE_NW(7); break;
      default: MACE_NW(8); break;
    }
#undef MACE_NW
  } else if (per_lane <= 8)
    launch_k(norm_kernel<8>, grid, 256, 0, s, x, ldx, rows, n_rows, d, W, B, layernorm, eps, O, ldo, rstd_out);
  else if (per_lane <= 24)
    launch_k(norm_kernel<24>, grid, 256, 0, s, x, ldx, rows, n_rows, d, W, B, layernorm, eps, O, ldo, rstd_out);
  else if (per_lane <= 64)
    launch_k(norm_kernel<64>, grid, 256, 0, s, x, ldx, rows, n_rows, d, W, B, layernorm, eps, O, ldo, rstd_out);
  else if (per_lane <= 128)
    launch_k(norm_kernel<128>, grid, 256, 0, s, x, ldx, rows, n_rows, d, W, B, layernorm, eps, O, ldo, rstd_out);
  else
    return mace_fail(ctx, MACE_ERR_ARG, "norm: d too large");
  ctx->launches++;
  return mace_check_launch(ctx, "norm");
}

extern "C" int mace_rope_kv(mace_ctx* ctx, void* qkv, int T, int Hq, int Hkv, int hd, const int* row_pos,
                            const int* row_seq, const int* row_kvi, const MaceSeq* seqs, const float* cos_t,
                            const float* sin_t, int apply_rope, const MaceKvLayout* kv, void* k_pool, void* v_pool,
                            void* stream) {
  if (T <= 0) return 0;
  if (hd % 16) return mace_fail(ctx, MACE_ERR_ARG, "rope_kv: hd % 16");
  launch_k(rope_kv_kernel, T, 128, 0, (cudaStream_t)stream, (__nv_bfloat16*)qkv, T, Hq, Hkv, hd, row_pos, row_seq, row_kvi,
                                                      seqs, cos_t, sin_t, apply_rope, *kv, (__nv_bfloat16*)k_pool,
                                                      (__nv_bfloat16*)v_pool);
  ctx->launches++;
  return mace_check_launch(ctx, "rope_kv");
}

extern "C" int mace_act(mace_ctx* ctx, const void* u, int T, int F, int swiglu, void* out, void* stream) {
  if (T <= 0) return 0;
  if (F % 8) return mace_fail(ctx, MACE_ERR_ARG, "act: F % 8");
  const size_t work = (size_t)T * F / 8;
  int grid = (int)((work + 255) / 256);
  if (grid > ctx->num_sms * 16) grid = ctx->num_sms * 16;
  launch_k(act_kernel, grid, 256, 0, (cudaStream_t)stream, (const __nv_bfloat16*)u, T, F, swiglu, (__nv_bfloat16*)out);
  ctx->launches++;
  return mace_check_launch(ctx, "act");
}

extern "C" int mace_argmax_keys(mace_ctx* ctx, unsigned long long* keys, int n, int* out, void* stream) {
  if (!ctx || (n > 0 && (!keys || !out))) return MACE_ERR_ARG;
  if (n <= 0) return 0;
  launch_k(argmax_keys_kernel, (n + 255) / 256, 256, 0, (cudaStream_t)stream, keys, n, out);
  ctx->launches++;
  return mace_check_launch(ctx, "argmax_keys");
}

extern "C" int mace_argmax(mace_ctx* ctx, const float* logits, int n, int V, int ld, int* out, void* stream) {
  if (n <= 0) return 0;
  launch_k(argmax_kernel, n, 1024, 0, (cudaStream_t)stream, logits, V, ld, out);
  ctx->launches++;
  return mace_check_launch(ctx, "argmax");
}
