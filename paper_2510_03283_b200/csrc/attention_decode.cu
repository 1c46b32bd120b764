// Paged decode attention (the HBM-bound hot kernel of decode-heavy ticks; reference stand-in:
// Engine._exec_decode's constant 20 ms charge, engine.py:592-594, plus the per-head windows of the
// prune trim, engine.py:506-511).
//
// Work item = (decode sequence, kv head, chunk of its page list); one WARP owns an item. The warp
// streams pages (16 tokens; a contiguous head-major K page + V page) through its private STAGES-deep
// cp.async.bulk ring (mbarrier transaction counts), so an SM keeps WARPS x STAGES x 2 pages in flight.
// Scores: lanes (t, half) each dot half of head_dim for token t and all G query heads of the GQA
// group (one K row read serves G heads), halves combine with one shuffle; then lanes own head_dim
// slices for P.V. Items are assigned to warps cyclically (static, deterministic); long contexts are
// split into chunks whose partial (m, l, acc) are merged in chunk order by the last finishing warp.
#include <cmath>

#include "common.cuh"
#include "mace_internal.h"

namespace mace {

// hd <= 64: 12 warps x 4-deep rings (C2 sweep on B200: 0.71 of HBM vs 0.68 for 16 x 3, 0.69 for 10 x 5,
// 0.57 for 8 x 6); hd 128: 8 warps x 3 (the 4 KB pages fill the smem budget)
#ifdef MACE_DEC_TRACE
__device__ unsigned long long* g_dec_trace = nullptr;  // [item][4]: start ns, end ns, pages, smid
#endif
#ifndef MACE_DEC2_WARPS64
#define MACE_DEC2_WARPS64 12  // sweep overrides (-D) for hd <= 64
#endif
#ifndef MACE_DEC2_STAGES64
#define MACE_DEC2_STAGES64 4
#endif
template <int HD, int G>
struct Dec2 {
  static constexpr int WARPS = HD >= 128 ? 8 : MACE_DEC2_WARPS64;
  static constexpr int STAGES = HD >= 128 ? 3 : MACE_DEC2_STAGES64;
  static constexpr int PAGE = kPageTokens * HD * 2;
  static constexpr int STAGE = 2 * PAGE;                      // K page | V page
  static constexpr int QH = HD / 2 + 4;                       // padded half row of q (bank spread)
  static constexpr int Q_OFF = STAGES * STAGE;                // fp32 [G][2][QH]
  static constexpr int P_OFF = Q_OFF + G * 2 * QH * 4;        // fp32 [16][G]
  static constexpr int BAR_OFF = P_OFF + 16 * G * 4;          // STAGES mbarriers
  static constexpr int WARP_BYTES = ((BAR_OFF + STAGES * 8) + 127) / 128 * 128;
  static constexpr int SMEM = WARPS * WARP_BYTES;
  static constexpr int DPL = HD / 32;                         // head dims per lane in P.V
  static constexpr int PARTIAL = 2 * G + G * HD;              // floats per chunk partial
};

template <int HD, int G>
__global__ void __launch_bounds__(Dec2<HD, G>::WARPS * 32) attn_decode2_kernel(
    const __nv_bfloat16* __restrict__ qkv, const MaceSeq* __restrict__ seqs, const int4* __restrict__ items,
    int n_items, const MaceKvLayout kv, const __nv_bfloat16* __restrict__ k_pool,
    const __nv_bfloat16* __restrict__ v_pool, int Hq, int Hkv, float scale_log2, __nv_bfloat16* __restrict__ out,
    float* __restrict__ head_norm, float* __restrict__ partials, int* __restrict__ counters,
    unsigned long long* __restrict__ work, unsigned long long n_warps_total) {
  using C = Dec2<HD, G>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ws = smem_raw + warp * C::WARP_BYTES;
  float* qs = reinterpret_cast<float*>(ws + C::Q_OFF);
  float* ps = reinterpret_cast<float*>(ws + C::P_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ws + C::BAR_OFF);
  if (lane == 0)
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[s], 1);
  fence_barrier_init();
  __syncwarp();
  pdl_wait();
  pdl_trigger();
  const int W = (Hq + 2 * Hkv) * HD;
  // lane (t, half) = (lane >> 1, lane & 1): each 8-lane phase of a 16-byte shared load covers 4 tokens x 2 halves,
  // and with the per-token chunk rotation below those are 8 distinct 4-bank groups (conflict-free K reads)
  const int t = lane >> 1, half = lane & 1;
  uint32_t ring_count = 0;  // pages issued by this warp so far (mbarrier phase bookkeeping across items)

  while (true) {
    // dynamic work distribution (items arrive longest-first) from a ticket counter that is zero between
    // launches: every warp draws exactly one ticket past the last item and leaves, so the warp drawing the
    // launch's final ticket (n_items + warps - 1) is the last to touch the counter and resets it
    unsigned long long ticket = 0;
    if (lane == 0) {
      ticket = atomicAdd(work, 1ull);
      if (ticket == (unsigned long long)n_items + n_warps_total - 1) atomicExch(work, 0ull);
    }
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    const long long item = (long long)ticket;
    if (item >= n_items) break;
    const int4 it = items[item];
    const MaceSeq sq = seqs[it.x];
    const int h = it.y, chunk = it.z >> 16, nch = it.z & 0xffff;
#ifdef MACE_DEC_TRACE
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
    // ---- q of the G query heads of this kv group -> fp32 smem
    const __nv_bfloat16* qrow = qkv + (size_t)sq.q_start * W + (size_t)h * G * HD;
    for (int i = lane; i < G * HD; i += 32) {
      const int g = i / HD, d = i % HD;
      qs[(g * 2 + d / (HD / 2)) * C::QH + d % (HD / 2)] = __bfloat162float(qrow[i]);
    }
    // ---- this chunk's pages: prompt pages split evenly, the last chunk adds the decode window
    const int n_pv = sq.n_pv;
    const int npp = (n_pv + 15) / 16;
    const int kvh = sq.slot * Hkv + h;
    const int d0 = kv.dec_first[kvh], db = kv.dec_base[kvh], de = kv.dec_end[sq.slot];
    const int r0 = (d0 - db) / 16;
    const int ndp = de > d0 ? ((de - 1 - db) / 16 - r0 + 1) : 0;
    const int per = (npp + nch - 1) / nch;
    const int s0 = min(npp, chunk * per);
    const int s1 = chunk == nch - 1 ? npp + ndp : min(npp, s0 + per);
    const int n_pg = s1 - s0;
    // page id + valid row range of every page slot of this chunk, one slot per lane register
    // (<= 96 slots: 32 prompt pages per chunk + the decode window), fetched once per item
    int pg_r[3], lh_r[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int p = s0 + lane + 32 * k;
      pg_r[k] = 0;
      lh_r[k] = 0;
      if (p < s1) {
        int lo, hi;
        if (p < npp) {
          pg_r[k] = kv.ptab[(size_t)sq.slot * kv.max_prompt_pages + p] * Hkv + h;
          lo = 0;
          hi = min(16, n_pv - 16 * p);
        } else {
          const int r = r0 + (p - npp);
          pg_r[k] = kv.dtab[(size_t)kvh * kv.max_dec_pages + r];
          const int b = db + 16 * r;
          lo = max(0, d0 - b);
          hi = min(16, de - b);
        }
        lh_r[k] = (lo << 8) | hi;
      }
    }
    auto slot_page = [&](int i) {
      const int v = i < 32 ? pg_r[0] : (i < 64 ? pg_r[1] : pg_r[2]);
      return __shfl_sync(0xffffffffu, v, i & 31);
    };
    auto slot_lohi = [&](int i) {
      const int v = i < 32 ? lh_r[0] : (i < 64 ? lh_r[1] : lh_r[2]);
      return __shfl_sync(0xffffffffu, v, i & 31);
    };
    auto issue = [&](int i, int pg, uint32_t count) {
      const int st = count % C::STAGES;
      uint8_t* dst = ws + st * C::STAGE;
      mbar_arrive_expect_tx(&bars[st], 2 * C::PAGE);
      bulk_load(dst, k_pool + (size_t)pg * 16 * HD, C::PAGE, &bars[st]);
      bulk_load(dst + C::PAGE, v_pool + (size_t)pg * 16 * HD, C::PAGE, &bars[st]);
    };
    __syncwarp();
    const uint32_t base_count = ring_count;
    for (int i = 0; i < n_pg && i < C::STAGES; ++i) {
      const int pg = slot_page(i);
      if (lane == 0) issue(i, pg, base_count + i);
    }
    float m[G], l[G], acc[G][C::DPL] __attribute__((aligned(8)));
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m[g] = -INFINITY;
      l[g] = 0.f;
#pragma unroll
      for (int d = 0; d < C::DPL; ++d) acc[g][d] = 0.f;
    }
    for (int i = 0; i < n_pg; ++i) {
      const uint32_t count = base_count + i;
      const int st = count % C::STAGES;
      mbar_wait(&bars[st], (count / C::STAGES) & 1);
      const uint8_t* stage = ws + st * C::STAGE;
      const int lh = slot_lohi(i);
      const int lo = lh >> 8, hi = lh & 0xff;
      const bool valid = t >= lo && t < hi;
      // ---- scores: lane (t, half) dots head dims [half*HD/2, (half+1)*HD/2) of token t, all G heads
      float2 sacc[G];
#pragma unroll
      for (int g = 0; g < G; ++g) sacc[g] = make_float2(0.f, 0.f);
      if (valid) {
        const __nv_bfloat16* krow = reinterpret_cast<const __nv_bfloat16*>(stage) + t * HD + half * (HD / 2);
        constexpr int NC = HD / 16;  // 16-byte chunks per half row
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          // rotate chunks across lanes so the 8 lanes of a load phase hit 8 distinct 4-bank groups (hd 128: the
          // two halves of a row are 32 words apart, i.e. the same banks, so they rotate apart too)
          const int cc = (HD >= 128 ? c + 2 * t + half : c + t) % NC;
          const uint4 u = *reinterpret_cast<const uint4*>(krow + cc * 8);
          const float2 k0 = bf2_to_f2(u.x), k1 = bf2_to_f2(u.y), k2 = bf2_to_f2(u.z), k3 = bf2_to_f2(u.w);
          const float* qh = qs + half * C::QH + cc * 8;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float4 qa = *reinterpret_cast<const float4*>(qh + g * 2 * C::QH);
            const float4 qb = *reinterpret_cast<const float4*>(qh + g * 2 * C::QH + 4);
            sacc[g] = ffma2(make_float2(qa.x, qa.y), k0, sacc[g]);
            sacc[g] = ffma2(make_float2(qa.z, qa.w), k1, sacc[g]);
            sacc[g] = ffma2(make_float2(qb.x, qb.y), k2, sacc[g]);
            sacc[g] = ffma2(make_float2(qb.z, qb.w), k3, sacc[g]);
          }
        }
      }
      // ---- online softmax per head over the page's 16 tokens (both half-lanes hold the same values)
      float alpha[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float sv = sacc[g].x + sacc[g].y;
        sv += __shfl_xor_sync(0xffffffffu, sv, 1);
        sv = valid ? sv * scale_log2 : -INFINITY;
        float mx = sv;
#pragma unroll
        for (int o = 16; o > 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float mn = fmaxf(m[g], mx);
        const float p = valid ? exp2f(sv - mn) : 0.f;
        float sum = p;
#pragma unroll
        for (int o = 16; o > 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        alpha[g] = (m[g] == -INFINITY) ? (mn == -INFINITY ? 1.f : 0.f) : exp2f(m[g] - mn);
        l[g] = l[g] * alpha[g] + sum;
        m[g] = mn;
        if (half == 0) ps[t * G + g] = p;
      }
      __syncwarp();
      // ---- P.V: lane owns DPL head dims; only the page's valid rows
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int d = 0; d < C::DPL; ++d) acc[g][d] *= alpha[g];
      const __nv_bfloat16* vpage = reinterpret_cast<const __nv_bfloat16*>(stage + C::PAGE);
      if (G == 1 && C::DPL == 2 && lo == 0 && hi == 16) {
        // full page (the common case): fully unrolled, two accumulator chains (even / odd tokens), p as float4
        float2 e = make_float2(acc[0][0], acc[0][1]), o = make_float2(0.f, 0.f);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 pw = *reinterpret_cast<const float4*>(ps + q4 * 4);
          const uint32_t* vr = reinterpret_cast<const uint32_t*>(vpage + (q4 * 4) * HD + lane * 2);
          const uint32_t w0 = vr[0], w1 = vr[HD / 2], w2 = vr[HD], w3 = vr[3 * HD / 2];
          e = ffma2(make_float2(pw.x, pw.x), bf2_to_f2(w0), e);
          o = ffma2(make_float2(pw.y, pw.y), bf2_to_f2(w1), o);
          e = ffma2(make_float2(pw.z, pw.z), bf2_to_f2(w2), e);
          o = ffma2(make_float2(pw.w, pw.w), bf2_to_f2(w3), o);
        }
        acc[0][0] = e.x + o.x;
        acc[0][C::DPL > 1 ? 1 : 0] = e.y + o.y;
      } else
#pragma unroll 4
      for (int tt = lo; tt < hi; ++tt) {
        float vv[C::DPL];
        if constexpr (C::DPL == 2) {
          const uint32_t w = *reinterpret_cast<const uint32_t*>(vpage + tt * HD + lane * 2);
          vv[0] = __uint_as_float(w << 16);
          vv[1] = __uint_as_float(w & 0xffff0000u);
        } else if constexpr (C::DPL == 4) {
          const uint2 w = *reinterpret_cast<const uint2*>(vpage + tt * HD + lane * 4);
          vv[0] = __uint_as_float(w.x << 16);
          vv[1] = __uint_as_float(w.x & 0xffff0000u);
          vv[2] = __uint_as_float(w.y << 16);
          vv[3] = __uint_as_float(w.y & 0xffff0000u);
        } else {
          vv[0] = __bfloat162float(vpage[tt * HD + lane]);
        }
        const float* prow = ps + tt * G;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float pw = prow[g];
          if constexpr (C::DPL >= 2) {
#pragma unroll
            for (int d = 0; d < C::DPL; d += 2) {
              const float2 r = ffma2(make_float2(pw, pw), make_float2(vv[d], vv[d + 1]), make_float2(acc[g][d], acc[g][d + 1]));
              acc[g][d] = r.x;
              acc[g][d + 1] = r.y;
            }
          } else {
            acc[g][0] = fmaf(pw, vv[0], acc[g][0]);
          }
        }
      }
      __syncwarp();
      if (i + C::STAGES < n_pg) {
        const int pg = slot_page(i + C::STAGES);
        if (lane == 0) issue(i + C::STAGES, pg, count + C::STAGES);
      }
    }
    ring_count = base_count + n_pg;
#ifdef MACE_DEC_TRACE
    if (g_dec_trace && lane == 0) {
      unsigned long long t_end, smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      asm volatile("{ .reg .u32 s; mov.u32 s, %%smid; cvt.u64.u32 %0, s; }" : "=l"(smid));
      g_dec_trace[item * 4 + 0] = t_start;
      g_dec_trace[item * 4 + 1] = t_end;
      g_dec_trace[item * 4 + 2] = n_pg;
      g_dec_trace[item * 4 + 3] = smid * 64 + warp;
    }
#endif

    // ---- epilogue: direct write (one chunk) or chunk partial + deterministic merge by the last warp
    const int row = sq.q_start;
    auto write_out = [&](const float* mm, const float* ll, float (*a)[C::DPL]) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float inv = ll[g] > 0.f ? 1.f / ll[g] : 0.f;
        float nrm = 0.f;
        __nv_bfloat16* o = out + (size_t)row * Hq * HD + (size_t)(h * G + g) * HD + lane * C::DPL;
#pragma unroll
        for (int d = 0; d < C::DPL; ++d) {
          const float v = a[g][d] * inv;
          o[d] = __float2bfloat16(v);
          nrm += v * v;
        }
        nrm = warp_sum(nrm);
        if (head_norm && lane == 0) head_norm[(size_t)row * Hq + h * G + g] = sqrtf(nrm);
      }
    };
    if (nch == 1) {
      write_out(m, l, acc);
      continue;
    }
    float* mine = partials + (size_t)(it.w + chunk) * C::PARTIAL;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (lane == 0) {
        mine[g] = m[g];
        mine[G + g] = l[g];
      }
#pragma unroll
      for (int d = 0; d < C::DPL; ++d) mine[2 * G + g * HD + lane * C::DPL + d] = acc[g][d];
    }
    __threadfence();
    __syncwarp();
    int prev = 0;
    if (lane == 0) prev = atomicAdd(&counters[kvh], 1);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != nch - 1) continue;
    __threadfence();
    const float* first = partials + (size_t)it.w * C::PARTIAL;
    float M[G], L[G], A[G][C::DPL];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      M[g] = -INFINITY;
      for (int c = 0; c < nch; ++c) M[g] = fmaxf(M[g], __ldcg(first + c * C::PARTIAL + g));
      L[g] = 0.f;
#pragma unroll
      for (int d = 0; d < C::DPL; ++d) A[g][d] = 0.f;
      for (int c = 0; c < nch; ++c) {  // chunk order: deterministic
        const float* pc = first + c * C::PARTIAL;
        const float mc = __ldcg(pc + g);
        const float sc = mc == -INFINITY ? 0.f : exp2f(mc - M[g]);
        L[g] += __ldcg(pc + G + g) * sc;
#pragma unroll
        for (int d = 0; d < C::DPL; ++d) A[g][d] += __ldcg(pc + 2 * G + g * HD + lane * C::DPL + d) * sc;
      }
    }
    write_out(M, L, A);
    if (lane == 0) counters[kvh] = 0;  // self-cleaning for the next launch
  }
}

template <int HD, int G>
int launch_decode2(MaceCtx* ctx, const MaceAttnArgs* a, float scale_log2, cudaStream_t s) {
  using C = Dec2<HD, G>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode2_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  const size_t need = (size_t)a->n_dec * C::PARTIAL * 4;
  if (!a->dec_workspace || a->dec_workspace_bytes < need || !a->dec_counters || !a->dec_work)
    return mace_fail(ctx, MACE_ERR_ARG, "attn decode: workspace/counters too small");
  const int per_sm = (227 * 1024) / C::SMEM;
  int grid = ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  const int need_ctas = (a->n_dec + C::WARPS - 1) / C::WARPS;
  if (grid > need_ctas) grid = need_ctas;
  // the kernel leaves the ticket counter at zero (its last ticket resets it): nothing to track here
  const unsigned long long base = (unsigned long long)grid * C::WARPS;
  launch_k(attn_decode2_kernel<HD, G>, grid, C::WARPS * 32, C::SMEM, s, 
      (const __nv_bfloat16*)a->qkv, a->seqs, reinterpret_cast<const int4*>(a->dec_items), a->n_dec, a->kv,
      (const __nv_bfloat16*)a->k_pool, (const __nv_bfloat16*)a->v_pool, a->Hq, a->Hkv, scale_log2,
      (__nv_bfloat16*)a->out, a->head_norm, (float*)a->dec_workspace, a->dec_counters, a->dec_work, base);
  ctx->launches++;
  return 0;
}

#ifdef MACE_DEC_TRACE
int dec_trace_set(void* buf) { return cudaMemcpyToSymbol(g_dec_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : -1; }
#endif

int dispatch_decode2(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s) {
  const int G = a->Hq / a->Hkv;
#define MACE_D2(HD_)                                                  \
  switch (G) {                                                        \
    case 1: return launch_decode2<HD_, 1>(ctx, a, sl2, s);            \
    case 2: return launch_decode2<HD_, 2>(ctx, a, sl2, s);            \
    case 4: return launch_decode2<HD_, 4>(ctx, a, sl2, s);            \
    case 8: return launch_decode2<HD_, 8>(ctx, a, sl2, s);            \
    default: return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn decode: GQA group must be 1, 2, 4 or 8"); \
  }
  switch (a->hd) {
    case 32: MACE_D2(32)
    case 64: MACE_D2(64)
    case 128: MACE_D2(128)
    default: return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn decode: head_dim must be 32, 64 or 128");
  }
#undef MACE_D2
}

}  // namespace mace

#ifdef MACE_DEC_TRACE
extern "C" int mace_debug_decode_trace(void* buf) { return mace::dec_trace_set(buf); }
#endif
