// Prefill / fine-tune attention, two query tiles per CTA (head_dim 64 / 128): the ping-pong form of
// attention.cu's attn_fa_kernel (same inputs, masks, outputs and LSE; reference stand-ins: Engine._exec_prefill
// engine.py:444-480 and the FT pair forward behind AlignmentEnv.pair_loss, alignment.py:151-166).
//
// Work item = (sequence, query head, PAIR of 128-row query blocks: A = block 2p, B = block 2p + 1). Every K / V
// tile is loaded once and serves both blocks. Roles (384 threads, one persistent CTA per SM):
//   warp 0      TMA: Q_A, Q_B (per item) and the K ring
//   warp 3      TMA: the V ring
//   warp 1      MMA issue (one elected lane), per KV tile j:
//                 S_A = Q_A K_j^T, S_B = Q_B K_j^T   (each once the P.V of that block's previous tile finished:
//                                                    P is written over S in TMEM)
//                 O_A += P_A V_j, O_B += P_B V_j     (A operand P read straight from TMEM)
//   warp 2      TMEM allocator (512 columns: S_A | S_B | O_A | O_B)
//   warps 4-7   softmax of block A, warps 8-11 softmax of block B: thread = one query row, all 128 scores of
//               the tile (no cross-warp row exchange); lazy rescale of O (only when the row max grows by > 2^8);
//               P packed to bf16 and stored over the first 64 columns of its S; epilogue O / l and the LSE.
// While one block's softmax runs on the CUDA cores, the tensor core works on the other block's S and P.V: the
// two softmax streams and the MMAs overlap instead of every tile's softmax latency sitting on the critical path.
#include <cmath>

#include "common.cuh"
#include "mace_internal.h"

namespace mace {

constexpr float kLog2eFa2 = 1.4426950408889634f;
constexpr float kRescaleLog2Fa2 = 8.f;  // lazy rescale threshold: p <= 2^8 between rescales (fp32-safe)
#ifndef MACE_FA2_EMU
#define MACE_FA2_EMU 0
#endif
constexpr int kEmuFa2 = MACE_FA2_EMU;
#ifndef MACE_FA2_F2FP
#define MACE_FA2_F2FP 0
#endif
constexpr bool kF2fpFa2 = MACE_FA2_F2FP;
#ifndef MACE_FA2_INORDER
#define MACE_FA2_INORDER 0
#endif
constexpr bool kInorderFa2 = MACE_FA2_INORDER;  // pack P with one F2FP (XU pipe) per pair instead of three ALU ops  // score pairs of every 8 exponentiated on the FMA pipe (A/B: tools/attn_bench.py)

template <int HD>
struct Fa2Cfg {
  static constexpr int SWZ = 128;
  static constexpr int ATOM = 64;
  static constexpr int KATOMS = HD / ATOM;
  static constexpr uint32_t LAYOUT = 2u;
  static constexpr int TILE = 128 * HD * 2;
  static constexpr int ATOM_BYTES = 128 * SWZ;
  static constexpr int ST = HD >= 128 ? 2 : 3;
  static constexpr int Q_OFF = 0;               // Q_A | Q_B
  static constexpr int KV_OFF = 2 * TILE;       // stage s: K at KV_OFF + 2s*TILE, V at + TILE
  static constexpr int BAR_OFF = KV_OFF + ST * 2 * TILE;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;
  static constexpr int S_COL = 0;               // S_A at 0, S_B at 128 (P_X over the first 64 columns of S_X)
  static constexpr int O_COL = 256;             // O_A at 256, O_B at 256 + HD
};

struct Fa2Item {
  MaceSeq sq;
  int hq, h, q0;   // q0: first query row of block A
  int n[2];        // KV tiles block A / B needs (0: block absent)
};
MACE_DEV Fa2Item fa2_item(const MaceSeq* seqs, const int4* items, int idx, int Hq, int Hkv) {
  const int4 it = items[idx];
  Fa2Item f;
  f.sq = seqs[it.x];
  f.hq = it.y;
  f.h = it.y / (Hq / Hkv);
  f.q0 = it.z * 256;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const int qs = f.q0 + 128 * b;
    f.n[b] = qs < f.sq.q_len ? (f.sq.kv_len - f.sq.q_len + min(qs + 127, f.sq.q_len - 1)) / 128 + 1 : 0;
  }
  return f;
}

template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_fa2_kernel(const __grid_constant__ TcMapsFa maps, const MaceSeq* __restrict__ seqs,
                    const int4* __restrict__ items, int n_items, const MaceKvLayout kv, int Hq, int Hkv,
                    float scale_log2, __nv_bfloat16* __restrict__ out, float* __restrict__ lse_out) {
  using C = Fa2Cfg<HD>;
  constexpr int ST = C::ST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* q_full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_empty = q_full + 1;
  uint64_t* k_full = q_empty + 1;    // [ST]
  uint64_t* k_empty = k_full + ST;   // [ST]
  uint64_t* v_full = k_empty + ST;   // [ST]
  uint64_t* v_empty = v_full + ST;   // [ST]
  uint64_t* s_full = v_empty + ST;   // [2] per block
  uint64_t* p_full = s_full + 2;     // [2]
  uint64_t* pv_done = p_full + 2;    // [2]
  uint64_t* o_free = pv_done + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 4);
      mbar_init(&pv_done[b], 1);
      mbar_init(&o_free[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------ producers: warp 0 Q + K, warp 3 V
    const bool is_k = warp == 0;
    pdl_wait();
    pdl_trigger();
    uint64_t* full = is_k ? k_full : v_full;
    uint64_t* empty = is_k ? k_empty : v_empty;
    const CUtensorMap* pool = is_k ? &maps.kpool : &maps.vpool;
    int g = 0;
    for (int idx = blockIdx.x, il = 0; idx < n_items; idx += gridDim.x, ++il) {
      const Fa2Item f = fa2_item(seqs, items, idx, Hq, Hkv);
      const bool dense = f.sq.kind == 2;
      if (is_k) {
        mbar_wait(q_empty, (il & 1) ^ 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(q_full, (f.n[1] ? 2 : 1) * C::TILE);
          for (int b = 0; b < (f.n[1] ? 2 : 1); ++b)
#pragma unroll
            for (int a = 0; a < C::KATOMS; ++a)
              tma_load_2d(smem + C::Q_OFF + b * C::TILE + a * C::ATOM_BYTES, &maps.q, q_full, f.hq * HD + a * C::ATOM,
                          f.sq.q_start + f.q0 + 128 * b);
        }
        __syncwarp();
      }
      const int n_kv = max(f.n[0], f.n[1]);
      const int maxp = (f.sq.kv_len + 15) / 16;
      const int* ptab_row = kv.ptab + (size_t)f.sq.slot * kv.max_prompt_pages;
      const int dense_col = (is_k ? Hq + f.h : Hq + Hkv + f.h) * HD;
      for (int j = 0; j < n_kv; ++j, ++g) {
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
    // ------------------------------------------------ MMA issuer. Order per KV tile j (anti-phase blocks):
    //   PV_A(j), [S_B(0) at j = 0], S_A(j+1), PV_B(j), S_B(j+1)
    // Block B starts half a period after A, so while one block's softmax runs the tensor core does the other
    // block's P.V and next S: the two softmax warpgroups alternate on the CUDA cores and the MMAs fill the gaps.
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t idesc_o = idesc_bf16_f32(128, HD, false, true);
    int c[2] = {0, 0};   // S / P.V issued per block so far (phases of s_full, p_full, pv_done)
    int u[2] = {0, 0};   // items that used O of each block (phase of o_free)
    int g0 = 0;          // CTA-global KV tile index of the item's tile 0
    auto issue_s = [&](int b, int st) {  // S_b = Q_b K^T into TMEM (P_b.V of the previous tile is done)
      // MACE_FA2_INORDER: rely on the single issuing thread's tcgen05.mma executing in issue order (P_b.V reads
      // the P columns before the next S_b writes them) instead of waiting for P_b.V's completion
      if (!kInorderFa2 && c[b] > 0) mbar_wait(&pv_done[b], (c[b] - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t qa = smem_u32(smem + C::Q_OFF + b * C::TILE);
        const uint32_t ka = smem_u32(smem + C::KV_OFF + 2 * st * C::TILE);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const int a = (k * 16) / C::ATOM, off = ((k * 16) % C::ATOM) * 2;
          umma_bf16(tmem + C::S_COL + 128 * b, smem_desc(qa + a * C::ATOM_BYTES + off, 16, 8 * C::SWZ, C::LAYOUT),
                    smem_desc(ka + a * C::ATOM_BYTES + off, 16, 8 * C::SWZ, C::LAYOUT), idesc_s, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[b]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int b, int j, int st) {  // O_b += P_b V (P read from TMEM)
      mbar_wait(&p_full[b], c[b] & 1);
      if (j == 0 && u[b] > 0) mbar_wait(&o_free[b], (u[b] - 1) & 1);  // the last item's epilogue read O_b
      tc_fence_after();
      if (elect_one()) {
        const uint32_t va = smem_u32(smem + C::KV_OFF + (2 * st + 1) * C::TILE);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          umma_bf16_ts(tmem + C::O_COL + HD * b, tmem + C::S_COL + 128 * b + k * 8,
                       smem_desc(va + k * 16 * C::SWZ, C::ATOM_BYTES, 8 * C::SWZ, C::LAYOUT), idesc_o,
                       (j > 0 || k > 0) ? 1u : 0u);
        umma_commit(&pv_done[b]);
      }
      __syncwarp();
      ++c[b];
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) umma_commit(bar);
      __syncwarp();
    };
    for (int idx = blockIdx.x, il = 0; idx < n_items; idx += gridDim.x, ++il) {
      const Fa2Item f = fa2_item(seqs, items, idx, Hq, Hkv);
      const int nA = f.n[0], nB = f.n[1], n_kv = max(nA, nB);
      auto stage = [&](int j) { return (g0 + j) % ST; };
      auto kwait = [&](int j) { mbar_wait(&k_full[stage(j)], ((g0 + j) / ST) & 1); };
      auto vwait = [&](int j) { mbar_wait(&v_full[stage(j)], ((g0 + j) / ST) & 1); };
      auto last_s = [&](int j) {  // after the last S that reads K(j): release it (and Q after the item's last S)
        commit(&k_empty[stage(j)]);
        if (j == n_kv - 1) commit(q_empty);
      };
      mbar_wait(q_full, il & 1);
      kwait(0);
      issue_s(0, stage(0));  // nA >= 1 always (block A is the pair's first block)
      if (nB == 0) last_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j < nA) {
          vwait(j);
          issue_pv(0, j, stage(j));
        }
        if (j == 0 && nB > 0) {
          issue_s(1, stage(0));
          last_s(0);
        }
        if (j + 1 < nA) {
          kwait(j + 1);
          issue_s(0, stage(j + 1));
          if (j + 1 >= nB) last_s(j + 1);
        }
        if (j < nB) {
          if (j >= nA) vwait(j);
          issue_pv(1, j, stage(j));
          if (j + 1 < nB) {
            if (j + 1 >= nA) kwait(j + 1);
            issue_s(1, stage(j + 1));
            last_s(j + 1);
          }
        }
        commit(&v_empty[stage(j)]);
      }
      g0 += n_kv;
#pragma unroll
      for (int b = 0; b < 2; ++b) u[b] += f.n[b] > 0;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue: block b = (warp - 4) / 4, thread = row
    pdl_wait();
    const int b = (warp - 4) >> 2;
    const int r = ((warp & 3) << 5) + lane;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t s_tm = tmem + C::S_COL + 128 * b + lane_base;
    const uint32_t o_tm = tmem + C::O_COL + HD * b + lane_base;
    int cnt = 0;  // tiles of this block processed (phases)
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
      const Fa2Item f = fa2_item(seqs, items, idx, Hq, Hkv);
      const int nt = f.n[b];
      if (nt == 0) continue;
      const int qi = f.q0 + 128 * b + r;
      const bool q_ok = qi < f.sq.q_len;
      const int lim_row = min(f.sq.kv_len - 1, f.sq.kv_len - f.sq.q_len + qi);
      const int h1 = f.sq.hole0 + f.sq.hole_len;
      const bool in_hole_rows = f.sq.kind == 2 && f.sq.hole_len > 0 && qi >= h1;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nt; ++j, ++cnt) {
        mbar_wait(&s_full[b], cnt & 1);
        tc_fence_after();
        uint32_t sv[128];
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_ld_32x32b_x32(s_tm + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(sv + 32 * q));
        tmem_ld_wait();
        const int lim = lim_row - j * 128;
        const int hlo = in_hole_rows ? f.sq.hole0 - j * 128 : 128, hhi = in_hole_rows ? h1 - j * 128 : 0;
        if (lim < 127 || (hlo < 128 && hhi > 0)) {  // causal diagonal / sequence end / pair hole -> -inf
#pragma unroll
          for (int cc = 0; cc < 128; ++cc)
            if (cc > lim || (cc >= hlo && cc < hhi)) sv[cc] = __float_as_uint(-INFINITY);
        }
        float mx8[8];  // row max: 8 independent chains of 3-input max (FMNMX3), 2 new scores per instruction
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = __uint_as_float(sv[i]);
#pragma unroll
        for (int cc = 8; cc < 120; cc += 16)
#pragma unroll
          for (int i = 0; i < 8; ++i) mx8[i] = fmax3(mx8[i], __uint_as_float(sv[cc + i]), __uint_as_float(sv[cc + 8 + i]));
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = fmaxf(mx8[i], __uint_as_float(sv[120 + i]));
        const float mx = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]));
        const float mx_s = mx * scale_log2;
        const bool grow = mx_s > m_run + kRescaleLog2Fa2;
        const float m_new = grow ? mx_s : m_run;
        const bool resc = grow && m_run != -INFINITY;
        const float alpha = resc ? exp2f(m_run - m_new) : 1.f;
        const float m_sub = m_new == -INFINITY ? 0.f : m_new;
        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_sub, -m_sub);
        const bool masked = lim < 127 || (hlo < 128 && hhi > 0) || m_new == -INFINITY;  // -inf scores: MUFU only
        float2 ps[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int cc = 0; cc < 128; cc += 2) {
          const float2 x = ffma2(make_float2(__uint_as_float(sv[cc]), __uint_as_float(sv[cc + 1])), sc2, nm2);
          // of every 8 score pairs, MACE_FA2_EMU on the FMA pipe (exp2_poly2) instead of MUFU (valid rows only)
          const float2 pv = (kEmuFa2 > 0 && !masked && ((cc >> 1) & 7) < kEmuFa2) ? exp2_poly2(x)
                                                                                  : make_float2(ex2_fast(x.x), ex2_fast(x.y));
          ps[(cc >> 1) & 3] = fadd2(ps[(cc >> 1) & 3], pv);
          sv[cc / 2] = kF2fpFa2 ? pack_bf16_cvt(pv.x, pv.y) : pack_bf16_alu(pv.x, pv.y);  // in place: pair cc/2
                                                                                         // overwrites consumed scores
        }
        const float2 pss = fadd2(fadd2(ps[0], ps[1]), fadd2(ps[2], ps[3]));
        l_run = l_run * alpha + (pss.x + pss.y);
        m_run = m_new;
        // P over S's first 64 columns (S_b(j) is in registers; P.V(j-1) finished before S_b(j) was issued)
        tmem_st_32x32b_x32(s_tm, *reinterpret_cast<const uint32_t(*)[32]>(sv));
        tmem_st_32x32b_x32(s_tm + 32, *reinterpret_cast<const uint32_t(*)[32]>(sv + 32));
        if (__any_sync(0xffffffffu, resc)) {  // resc implies j >= 1: O holds P.V up to tile j-1 (complete)
#pragma unroll 1
          for (int c0 = 0; c0 < HD; c0 += 16) {
            uint32_t o[16];
            tmem_ld_32x32b_x16(o_tm + c0, o);
            tmem_ld_wait();
#pragma unroll
            for (int cc = 0; cc < 16; ++cc) o[cc] = __float_as_uint(__uint_as_float(o[cc]) * alpha);
            tmem_st_32x32b_x16(o_tm + c0, o);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
      }
      // ---- epilogue: O / l -> bf16 rows, LSE; then O_b is free for the next item
      mbar_wait(&pv_done[b], (cnt - 1) & 1);
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      __nv_bfloat16* o_row = out + (size_t)(f.sq.q_start + qi) * Hq * HD + f.hq * HD;
#pragma unroll 1
      for (int c0 = 0; c0 < HD; c0 += 16) {
        uint32_t o[16];
        tmem_ld_32x32b_x16(o_tm + c0, o);
        tmem_ld_wait();
        if (q_ok) {
#pragma unroll
          for (int cc = 0; cc < 16; cc += 8) {
            const uint4 v = make_uint4(pack_bf16(__uint_as_float(o[cc]) * inv, __uint_as_float(o[cc + 1]) * inv),
                                       pack_bf16(__uint_as_float(o[cc + 2]) * inv, __uint_as_float(o[cc + 3]) * inv),
                                       pack_bf16(__uint_as_float(o[cc + 4]) * inv, __uint_as_float(o[cc + 5]) * inv),
                                       pack_bf16(__uint_as_float(o[cc + 6]) * inv, __uint_as_float(o[cc + 7]) * inv));
            *reinterpret_cast<uint4*>(o_row + c0 + cc) = v;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[b]);
      if (q_ok && lse_out) lse_out[(size_t)(f.sq.q_start + qi) * Hq + f.hq] = (m_run + log2f(l_run)) / kLog2eFa2;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// host: tensor maps exactly as the single-tile kernel (qkv rows for Q and dense K / V, head-major page pools)
template <int HD>
int launch_fa2(MaceCtx* ctx, const MaceAttnArgs* a, float scale_log2, cudaStream_t s, const TcMapsFa& maps) {
  using C = Fa2Cfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_fa2_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  launch_k(attn_fa2_kernel<HD>, a->n_tc < ctx->num_sms ? a->n_tc : ctx->num_sms, 384, C::SMEM, s, maps, a->seqs,
           reinterpret_cast<const int4*>(a->tc_items), a->n_tc, a->kv, a->Hq, a->Hkv, scale_log2,
           (__nv_bfloat16*)a->out, a->lse);
  ctx->launches++;
  return 0;
}
template int launch_fa2<64>(MaceCtx*, const MaceAttnArgs*, float, cudaStream_t, const TcMapsFa&);
template int launch_fa2<128>(MaceCtx*, const MaceAttnArgs*, float, cudaStream_t, const TcMapsFa&);

}  // namespace mace
