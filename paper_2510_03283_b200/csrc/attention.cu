// Ragged paged attention forward for the hybrid iteration: prefill, decode and fine-tune sequences of
// one tick in one call (reference stand-ins replaced: Engine._exec_prefill engine.py:444-480,
// Engine._exec_decode engine.py:482-532, the FT pair forward behind AlignmentEnv.pair_loss
// alignment.py:151-166).
//
//  * tc path (prefill + fine-tune sequences, tensor-core bound): attn_fa_kernel below (persistent,
//    warp-specialised, S and O accumulators and P all in TMEM). Paged K/V come from the head-major page
//    pools, dense FT K/V straight from the packed qkv rows.
//  * decode path (HBM bound): attention_decode.cu (warp per (sequence, kv head, chunk) item).
#include <cmath>

#include "common.cuh"
#include "mace_internal.h"

namespace mace {

constexpr float kLog2e = 1.4426950408889634f;

using TcMaps = TcMapsFa;  // mace_internal.h
template <int HD>
int launch_fa2(MaceCtx* ctx, const MaceAttnArgs* a, float scale_log2, cudaStream_t s, const TcMapsFa& maps);

// =====================================================================================================
// warp-specialised tensor-core path
//
// Persistent CTA (one per SM) over 128-query-row x 1-head items, 384 threads:
//   warp 0      TMA producer of Q (double-buffered by item) and K tiles of 128 keys (ST-stage ring; page
//               ids fetched by 8 lanes in parallel, one TMA box per 16-token page and swizzle atom)
//   warp 3      TMA producer of V tiles (own ring: K_j is released when S(j) completes, V_j after P(j).V_j)
//   warp 1      MMA issuer (one elected lane): S(g+1) = Q K^T as soon as the softmax has pulled S(g) out of
//               TMEM, then O += P(g) V_g with P read from TMEM (tcgen05.mma A-from-TMEM: no smem round trip)
//   warp 2      TMEM allocator: S fp32 | P bf16 | O x 2 (item parity) | row-stat exchange columns
//   warps 4..11 softmax: two warpgroups split every row's 128 scores (WG0 keys 0-63, WG1 64-127), row max
//               exchanged through TMEM; exp2 with a lazily updated running max (O in TMEM is rescaled only
//               when the max grows by > 2^8); P packed to bf16 on the ALU and stored to TMEM; epilogue O/l.
// Measured (tools/attn_bench.py, tools/attn_trace.py): ~790 TF/s at hd 128, ~480 at hd 64 on B200; the
// softmax warps are the critical path (exp phase ~1400 of ~2900 cycles per tile, the rest latency).
// =====================================================================================================
template <int HD>
struct FaCfg {
  static constexpr int SWZ = HD >= 64 ? 128 : 64;
  static constexpr int ATOM = SWZ / 2;
  static constexpr int KATOMS = HD / ATOM;
  static constexpr uint32_t LAYOUT = SWZ == 128 ? 2u : 4u;
  static constexpr int TILE = 128 * HD * 2;
  static constexpr int ATOM_BYTES = 128 * SWZ;
  static constexpr int ST = HD >= 128 ? 2 : 3;
  static constexpr int Q_OFF = 0;                     // 2 buffers (item parity)
  static constexpr int KV_OFF = 2 * TILE;             // stage s: K at KV_OFF + 2s*TILE, V at +TILE
  static constexpr int BAR_OFF = KV_OFF + ST * 2 * TILE;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  // TMEM: S fp32 (128 cols) | P bf16x2 (64 cols: the A operand of P.V, never in smem) | O (item parity,
  // 2 x HD) | 6 exchange columns of the two softmax WGs (row max, row sum)
  static constexpr int P_COL = 128;
  static constexpr int O_COL = 192;
  static constexpr int XCOL = O_COL + 2 * HD;
  static constexpr int TMEM_COLS = XCOL + 8 <= 256 ? 256 : 512;
};
constexpr float kRescaleLog2 = 8.f;  // lazy rescale threshold: p <= 2^8 between rescales (fp32-safe)
#ifndef MACE_EMU_PAIRS
#define MACE_EMU_PAIRS 0
#endif
// of every 8 score pairs, exp2 on the FMA pipe. Measured on B200 (tools/attn_bench.py, tools/attn_trace.py):
// the two softmax warpgroups are latency/issue-bound, not MUFU-bound, so every emulated pair is slower; 0.
constexpr int kEmuPairs = MACE_EMU_PAIRS;

struct FaItem {
  MaceSeq sq;
  int hq, h, q0, n_tiles;
};
MACE_DEV FaItem fa_item(const MaceSeq* seqs, const int4* items, int idx, int Hq, int Hkv) {
  const int4 it = items[idx];
  FaItem f;
  f.sq = seqs[it.x];
  f.hq = it.y;
  f.h = it.y / (Hq / Hkv);
  f.q0 = it.z * 128;
  const int q_last_log = f.sq.kv_len - f.sq.q_len + min(f.q0 + 127, f.sq.q_len - 1);
  f.n_tiles = q_last_log / 128 + 1;
  return f;
}

#ifdef MACE_ATTN_TRACE
__device__ long long* g_attn_trace = nullptr;  // [role 3][event 8][tile 64] clock64 of CTA 0
#define ATR(role, ev, g)                                                                        \
  do {                                                                                          \
    if (g_attn_trace && blockIdx.x == 0 && (g) < 64) g_attn_trace[((role) * 8 + (ev)) * 64 + (g)] = clock64(); \
  } while (0)
#else
#define ATR(role, ev, g)
#endif

// Persistent: CTA b walks items b, b + grid, ... of the longest-first item list. Every role walks the same
// (item, KV tile) sequence with a CTA-global tile counter g for the ring phases; Q and O are double
// buffered by item parity so the next item's loads / first S overlap this item's last softmax and epilogue.
template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_fa_kernel(const __grid_constant__ TcMaps maps, const MaceSeq* __restrict__ seqs, const int4* __restrict__ items,
                   int n_items, const MaceKvLayout kv, int Hq, int Hkv, float scale_log2,
                   __nv_bfloat16* __restrict__ out, float* __restrict__ lse_out) {
  using C = FaCfg<HD>;
  constexpr int ST = C::ST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* q_full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);  // [2]
  uint64_t* q_empty = q_full + 2;      // [2]
  uint64_t* k_full = q_empty + 2;      // [ST]
  uint64_t* k_empty = k_full + ST;     // [ST]
  uint64_t* v_full = k_empty + ST;     // [ST]
  uint64_t* v_empty = v_full + ST;     // [ST]
  uint64_t* s_full = v_empty + ST;
  uint64_t* s_free = s_full + 1;
  uint64_t* p_full = s_free + 1;       // [2]
  uint64_t* o_done = p_full + 2;       // [2]
  uint64_t* o_free = o_done + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&p_full[s], 8);
      mbar_init(&o_done[s], 1);
      mbar_init(&o_free[s], 8);
    }
    for (int s = 0; s < ST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 8);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_s = tmem;

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------ producers: warp 0 streams Q and K, warp 3 streams V
    const bool is_k = warp == 0;
    pdl_wait();
    pdl_trigger();
    uint64_t* full = is_k ? k_full : v_full;
    uint64_t* empty = is_k ? k_empty : v_empty;
    const CUtensorMap* pool = is_k ? &maps.kpool : &maps.vpool;
    int g = 0;
    for (int idx = blockIdx.x, il = 0; idx < n_items; idx += gridDim.x, ++il) {
      const FaItem f = fa_item(seqs, items, idx, Hq, Hkv);
      const bool dense = f.sq.kind == 2;
      if (is_k) {
        const int qb = il & 1;
        mbar_wait(&q_empty[qb], ((il >> 1) & 1) ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&q_full[qb], C::TILE);
#pragma unroll
          for (int a = 0; a < C::KATOMS; ++a)
            tma_load_2d(smem + C::Q_OFF + qb * C::TILE + a * C::ATOM_BYTES, &maps.q, &q_full[qb],
                        f.hq * HD + a * C::ATOM, f.sq.q_start + f.q0);
        }
        __syncwarp();
      }
      const int maxp = (f.sq.kv_len + 15) / 16;
      const int* ptab_row = kv.ptab + (size_t)f.sq.slot * kv.max_prompt_pages;
      const int dense_col = (is_k ? Hq + f.h : Hq + Hkv + f.h) * HD;
      for (int j = 0; j < f.n_tiles; ++j, ++g) {
        const int st = g % ST;
        int pg = 0;
        if (!dense && lane < 8) pg = ptab_row[min(j * 8 + lane, maxp - 1)] * Hkv + f.h;
        mbar_wait(&empty[st], ((g / ST) & 1) ^ 1);
        uint8_t* dst = smem + C::KV_OFF + (2 * st + (is_k ? 0 : 1)) * C::TILE;
        if (lane == 0) mbar_arrive_expect_tx(&full[st], C::TILE);
        if (dense) {
          if (lane == 0) {
#pragma unroll
            for (int a = 0; a < C::KATOMS; ++a)
              tma_load_2d(dst + a * C::ATOM_BYTES, &maps.q, &full[st], dense_col + a * C::ATOM, f.sq.q_start + j * 128);
          }
        } else {
#pragma unroll
          for (int ps = 0; ps < 8; ++ps) {
            const int page = __shfl_sync(0xffffffffu, pg, ps);
            if (lane == 0) {
#pragma unroll
              for (int a = 0; a < C::KATOMS; ++a)
                tma_load_2d(dst + a * C::ATOM_BYTES + ps * 16 * C::SWZ, pool, &full[st], a * C::ATOM, page * 16);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(128, HD, false, true);
    // S(g) = Q K_g^T once the softmax has pulled S(g-1) into registers (K_g resident)
    auto issue_s = [&](int g, int qb, bool last_of_item) {
      const int st = g % ST;
      mbar_wait(&k_full[st], (g / ST) & 1);
      if (g > 0) mbar_wait(s_free, (g - 1) & 1);
      tc_fence_after();
      if (lane == 0) ATR(2, 0, g);
      if (elect_one()) {
        const uint32_t qa = smem_u32(smem + C::Q_OFF + qb * C::TILE);
        const uint32_t ka = smem_u32(smem + C::KV_OFF + 2 * st * C::TILE);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const int a = (k * 16) / C::ATOM, off = ((k * 16) % C::ATOM) * 2;
          umma_bf16(tmem_s, smem_desc(qa + a * C::ATOM_BYTES + off, 16, 8 * C::SWZ, C::LAYOUT),
                    smem_desc(ka + a * C::ATOM_BYTES + off, 16, 8 * C::SWZ, C::LAYOUT), idesc_s, k > 0 ? 1u : 0u);
        }
        umma_commit(s_full);
        umma_commit(&k_empty[st]);
        if (last_of_item) umma_commit(&q_empty[qb]);
      }
      __syncwarp();
    };
    int g = 0;
    for (int idx = blockIdx.x, il = 0; idx < n_items; idx += gridDim.x, ++il) {
      const FaItem f = fa_item(seqs, items, idx, Hq, Hkv);
      const int qb = il & 1, ob = il & 1;
      const uint32_t tmem_o = tmem + C::O_COL + ob * HD;
      mbar_wait(&q_full[qb], (il >> 1) & 1);
      for (int j = 0; j < f.n_tiles; ++j, ++g) {
        if (j == 0) issue_s(g, qb, f.n_tiles == 1);
        if (j + 1 < f.n_tiles) issue_s(g + 1, qb, j + 2 == f.n_tiles);
        mbar_wait(&v_full[g % ST], (g / ST) & 1);
        mbar_wait(&p_full[g & 1], (g >> 1) & 1);
        if (j == 0) mbar_wait(&o_free[ob], ((il >> 1) & 1) ^ 1);  // epilogue of item il-2 has read this O
        tc_fence_after();
        if (lane == 0) ATR(2, 1, g);
        if (elect_one()) {
          const uint32_t va = smem_u32(smem + C::KV_OFF + 2 * (g % ST) * C::TILE + C::TILE);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            umma_bf16_ts(tmem_o, tmem + C::P_COL + k * 8,
                         smem_desc(va + k * 16 * C::SWZ, C::ATOM_BYTES, 8 * C::SWZ, C::LAYOUT), idesc_o,
                         (j > 0 || k > 0) ? 1u : 0u);
          umma_commit(&o_done[g & 1]);
          umma_commit(&v_empty[g % ST]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue: two warpgroups split every row's 128
    // scores (WG0 columns 0-63, WG1 64-127; warps 4+k and 8+k own TMEM lanes 32k..32k+31). Two warps per
    // SMSP hide the exp / FFMA latencies one warp cannot; the row max is exchanged through smem.
    pdl_wait();
    const int wg = (warp - 4) >> 2;
    const int r = ((warp & 3) << 5) + lane;
    const int cb = wg * 64;
    const uint32_t pair_bar = 1 + (warp & 3);  // named barrier of warps (4+k, 8+k)
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t xcol = tmem + C::XCOL + lane_base;  // this warp's lanes of the exchange columns
    const uint32_t p_tm = tmem + C::P_COL + lane_base + wg * 32;  // this WG's 64 keys of P (32 columns)
    int g = 0;
    for (int idx = blockIdx.x, il = 0; idx < n_items; idx += gridDim.x, ++il) {
      const FaItem f = fa_item(seqs, items, idx, Hq, Hkv);
      const uint32_t tmem_o = tmem + C::O_COL + (il & 1) * HD + wg * (HD / 2);
      const int qi = f.q0 + r;
      const bool q_ok = qi < f.sq.q_len;
      const int lim_row = min(f.sq.kv_len - 1, f.sq.kv_len - f.sq.q_len + qi);  // last visible key of this row
      // FT preference pair (MaceSeq hole): the rejected branch's rows do not see the chosen branch's keys
      const int h1 = f.sq.hole0 + f.sq.hole_len;
      const bool in_hole_rows = f.sq.kind == 2 && f.sq.hole_len > 0 && qi >= h1;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < f.n_tiles; ++j, ++g) {
        mbar_wait(s_full, g & 1);
        tc_fence_after();
        if (lane == 0) ATR(wg, 0, g);
        uint32_t sv[64];
        tmem_ld_32x32b_x32(tmem_s + lane_base + cb, *reinterpret_cast<uint32_t(*)[32]>(sv));
        tmem_ld_32x32b_x32(tmem_s + lane_base + cb + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
        if (lane == 0) ATR(wg, 1, g);
        const int lim = lim_row - j * 128 - cb;
        const int hlo = in_hole_rows ? f.sq.hole0 - j * 128 - cb : 64, hhi = in_hole_rows ? h1 - j * 128 - cb : 0;
        if (lim < 63 || (hlo < 64 && hhi > 0)) {  // causal diagonal / sequence end / pair hole: masked -> -inf
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c > lim || (c >= hlo && c < hhi)) sv[c] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = __uint_as_float(sv[i]);
#pragma unroll
        for (int c = 8; c < 64; c += 16) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            mx8[i] = fmaxf(mx8[i], fmaxf(__uint_as_float(sv[c + i]), c + 8 + i < 64 ? __uint_as_float(sv[c + 8 + i]) : -INFINITY));
        }
        const float mxp = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        // exchange through TMEM (same lanes, spare columns; parity-double-buffered so one barrier suffices)
        tmem_st_x1(xcol + (g & 1) * 2 + wg, __float_as_uint(mxp));
        tmem_st_wait();
        tc_fence_before();
        named_bar_sync(pair_bar, 64);
        tc_fence_after();
        const float mx = fmaxf(mxp, __uint_as_float(tmem_ld_x1(xcol + (g & 1) * 2 + (wg ^ 1))));
        tmem_ld_wait();
        if (lane == 0) ATR(wg, 2, g);
        const float mx_s = mx * scale_log2;
        const bool grow = mx_s > m_run + kRescaleLog2;
        const float m_new = grow ? mx_s : m_run;
        const bool resc = grow && m_run != -INFINITY;
        const float alpha = resc ? exp2f(m_run - m_new) : 1.f;
        const float m_sub = m_new == -INFINITY ? 0.f : m_new;  // fully masked row so far: p = exp2(-inf) = 0
        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_sub, -m_sub);
        float2 ps[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const bool emu = kEmuPairs > 0 && lim >= 63 && m_new != -INFINITY;
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float2 x = ffma2(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sc2, nm2);
          const float2 pv = (emu && ((c >> 1) & 7) < kEmuPairs) ? exp2_poly2(x)
                                                                 : make_float2(ex2_fast(x.x), ex2_fast(x.y));
          ps[(c >> 1) & 3] = fadd2(ps[(c >> 1) & 3], pv);
          sv[c / 2] = pack_bf16_alu(pv.x, pv.y);  // in place: pair c/2 only overwrites consumed scores
        }
        const float2 pss = fadd2(fadd2(ps[0], ps[1]), fadd2(ps[2], ps[3]));
        l_run = l_run * alpha + (pss.x + pss.y);
        m_run = m_new;
        if (lane == 0) ATR(wg, 3, g);
        // the single P buffer was read by PV(g-1), which also completed O up to tile j-1
        if (g >= 1) mbar_wait(&o_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
        if (lane == 0) ATR(wg, 4, g);
        tmem_st_32x32b_x32(p_tm, *reinterpret_cast<const uint32_t(*)[32]>(sv));
        if (__any_sync(0xffffffffu, resc)) {  // resc implies j >= 1: O holds this item's PV up to j-1
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < HD / 2; c0 += 16) {
            uint32_t o[16];
            tmem_ld_32x32b_x16(tmem_o + lane_base + c0, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 16; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
            tmem_st_32x32b_x16(tmem_o + lane_base + c0, o);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g & 1]);
        if (lane == 0) ATR(wg, 5, g);
      }
      // ---- epilogue of the item: this WG's HD/2 columns of O / l -> bf16, LSE; then the O buffer is free
      tmem_st_x1(xcol + 4 + wg, __float_as_uint(l_run));
      tmem_st_wait();
      tc_fence_before();
      named_bar_sync(pair_bar, 64);
      tc_fence_after();
      const float l_tot = l_run + __uint_as_float(tmem_ld_x1(xcol + 4 + (wg ^ 1)));
      tmem_ld_wait();
      mbar_wait(&o_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
      tc_fence_after();
      const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
      __nv_bfloat16* o_row = out + (size_t)(f.sq.q_start + qi) * Hq * HD + f.hq * HD + wg * (HD / 2);
#pragma unroll 1
      for (int c0 = 0; c0 < HD / 2; c0 += 16) {
        uint32_t o[16];
        tmem_ld_32x32b_x16(tmem_o + lane_base + c0, o);
        tmem_ld_wait();
        if (q_ok) {
#pragma unroll
          for (int c = 0; c < 16; c += 8) {
            const uint4 v = make_uint4(pack_bf16(__uint_as_float(o[c]) * inv, __uint_as_float(o[c + 1]) * inv),
                                       pack_bf16(__uint_as_float(o[c + 2]) * inv, __uint_as_float(o[c + 3]) * inv),
                                       pack_bf16(__uint_as_float(o[c + 4]) * inv, __uint_as_float(o[c + 5]) * inv),
                                       pack_bf16(__uint_as_float(o[c + 6]) * inv, __uint_as_float(o[c + 7]) * inv));
            *reinterpret_cast<uint4*>(o_row + c0 + c) = v;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[il & 1]);
      if (wg == 0 && q_ok && lse_out)
        lse_out[(size_t)(f.sq.q_start + qi) * Hq + f.hq] = (m_run + log2f(l_tot)) / kLog2e;
      named_bar_sync(pair_bar, 64);  // the row-sum columns are rewritten by the next item's epilogue
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

// =====================================================================================================
// host
// =====================================================================================================
static bool encode_2d(MaceCtx* ctx, CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                      uint32_t box_inner, uint32_t box_outer, int swz_bytes) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swz_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  return ctx->encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD>
static int launch_tc(MaceCtx* ctx, const MaceAttnArgs* a, float scale_log2, cudaStream_t s) {
  using C = FaCfg<HD>;
  TcMaps maps;
  const int W = (a->Hq + 2 * a->Hkv) * HD;
  bool ok = encode_2d(ctx, &maps.q, a->qkv, W, a->T, W, C::ATOM, 128, C::SWZ);
  const void* kp = a->k_pool ? a->k_pool : a->qkv;
  const void* vp = a->v_pool ? a->v_pool : a->qkv;
  const uint64_t rows = a->k_pool ? (uint64_t)a->pool_pages * 16 : (uint64_t)a->T;
  const uint64_t ld = a->k_pool ? HD : W;
  ok = ok && encode_2d(ctx, &maps.kpool, kp, HD, rows, ld, C::ATOM, 16, C::SWZ) &&
       encode_2d(ctx, &maps.vpool, vp, HD, rows, ld, C::ATOM, 16, C::SWZ);
  if (!ok) return mace_fail(ctx, MACE_ERR_LAUNCH, "attn: tensor map encode failed");
  if constexpr (HD == 64 || HD == 128) {
    if (a->tc_pairs) return launch_fa2<HD>(ctx, a, scale_log2, s, maps);  // items are query-block pairs
  } else {
    if (a->tc_pairs) return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn: query-block pair items need head_dim 64 / 128");
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_fa_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, FaCfg<HD>::SMEM);
    attr = true;
  }
  launch_k(attn_fa_kernel<HD>, a->n_tc < ctx->num_sms ? a->n_tc : ctx->num_sms, 384, FaCfg<HD>::SMEM, s, maps,
           a->seqs, reinterpret_cast<const int4*>(a->tc_items), a->n_tc, a->kv, a->Hq, a->Hkv, scale_log2,
           (__nv_bfloat16*)a->out, a->lse);
  ctx->launches++;
  return 0;
}

int dispatch_decode2(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s);
int dispatch_decode_tc(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s);

}  // namespace mace

using namespace mace;

#ifdef MACE_ATTN_TRACE
extern "C" int mace_debug_attn_trace(void* buf) {
  return cudaMemcpyToSymbol(mace::g_attn_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int mace_attn_fwd(mace_ctx* ctx, const MaceAttnArgs* a, void* stream) {
  if (!ctx || !a) return MACE_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const float scale = a->scale > 0.f ? a->scale : 1.f / sqrtf((float)a->hd);
  const float sl2 = scale * kLog2e;
  if (a->Hq % a->Hkv) return mace_fail(ctx, MACE_ERR_ARG, "attn: Hq % Hkv");
  int rc = 0;
  if (a->n_tc > 0) {
    switch (a->hd) {
      case 32: rc = launch_tc<32>(ctx, a, sl2, s); break;
      case 64: rc = launch_tc<64>(ctx, a, sl2, s); break;
      case 128: rc = launch_tc<128>(ctx, a, sl2, s); break;
      default: return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn: head_dim must be 32, 64 or 128");
    }
    if (rc) return rc;
  }
  if (a->n_dec > 0) {
    if (!a->k_pool || !a->v_pool) return mace_fail(ctx, MACE_ERR_ARG, "attn: decode rows need KV pools");
    // auto: GQA groups (G >= 2) run on the tcgen05 swap-AB kernel (the CUDA-core kernel is issue-bound
    // there, G dots per K row); plain MHA (G = 1) keeps the CUDA-core streaming kernel (measured faster)
    const int impl = a->decode_impl ? a->decode_impl : (a->Hq / a->Hkv >= 2 ? 2 : 1);
    rc = impl == 1 ? dispatch_decode2(ctx, a, sl2, s) : dispatch_decode_tc(ctx, a, sl2, s);
    if (rc) return rc;
  }
  return mace_check_launch(ctx, "attn_fwd");
}
