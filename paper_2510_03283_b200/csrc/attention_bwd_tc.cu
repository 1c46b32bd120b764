// Attention backward on tcgen05 for the fine-tune rows (dense causal FT sequences), head_dim 64 / 128.
//
// Reference stand-in replaced: the DPO step behind AlignmentEnv.ft_step (alignment.py:168-172) backpropagates
// through the selected layers; this is the attention core of that backward (FT rows only).
//
// CTA = one key block (128 keys) of one KV head; it walks every (query head of the GQA group, query block at
// or after the key block) step and keeps dK, dV in TMEM for the whole walk. Warps 0-3 compute (thread r = TMEM
// lane r), warp 4 issues TMA and MMA; they hand off through mbarriers. Per step (Q_i, dO_i double-buffered by
// TMA, the next step's tiles load during this one):
//   S^T  = K Q^T,  dP^T = V dO^T                      (tcgen05, keys on lanes, queries as N)
//   P^T  = exp2(S^T * scale*log2e - lse2[q]) (causal), dS^T = P^T (dP^T - D[q])   (thread = key row)
//   P^T -> TMEM (bf16, A operand), dS -> smem (one bf16 tile read twice: K-major for dK, MN-major for dQ)
//   dV  += P^T dO   (A from TMEM),  dK += dS^T Q,  dQ = dS K  (queries on lanes) -> red.global.add.v4 into
//   the fp32 dQ rows (several key blocks and GQA heads contribute), dK / dV written once at the end.
#include <cmath>

#include "common.cuh"
#include "mace_internal.h"

namespace mace {

template <int HD>
struct BwdCfg {
  static constexpr int SWZ = 128;
  static constexpr int ATOM = 64;                   // bf16 per 128-byte swizzle row
  static constexpr int KATOMS = HD / ATOM;
  static constexpr int TILE = 128 * HD * 2;         // one 128-row tile
  static constexpr int ATOM_BYTES = 128 * SWZ;      // 128 rows x 128 B
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = TILE;
  static constexpr int QD_OFF = 2 * TILE;           // buffer b: Q at QD_OFF + 2b*TILE, dO at +TILE
  static constexpr int DS_OFF = 6 * TILE;           // dS [128 keys][128 queries] bf16, 128B swizzle
  static constexpr int LD_OFF = DS_OFF + 128 * 128 * 2;  // lse * log2e [128], D [128] of the step's queries
  static constexpr int BAR_OFF = LD_OFF + 2 * 128 * 4;
  static constexpr int SMEM = BAR_OFF + 128 + 1024;
  static constexpr uint32_t COL_S = 0, COL_P = 128, COL_DV = 256, COL_DK = 256 + HD;  // TMEM (dQ reuses COL_S)
};

MACE_DEV void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

struct BwdMaps {
  CUtensorMap qkv;   // [T, W] bf16, box {64, 128}
  CUtensorMap dout;  // [T, Hq*HD] bf16, box {64, 128}
};

template <int HD>
__global__ void __launch_bounds__(160, 1)
    attn_bwd_tc_kernel(const __grid_constant__ BwdMaps maps, const float* __restrict__ lse,
                       const float* __restrict__ Dv, const MaceSeq* __restrict__ seqs, const int4* __restrict__ items,
                       int Hq, int Hkv, float scale, float* __restrict__ dqkv, int row_offset,
                       int* __restrict__ dq_order) {
  using C = BwdCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* qd_full = kv_full + 1;  // [2]
  uint64_t* sp_done = kv_full + 3;  // S^T, dP^T in TMEM                      (MMA -> compute)
  uint64_t* ds_ready = kv_full + 4; // P^T in TMEM, dS in smem               (compute -> MMA, 4 warps)
  uint64_t* mm_done = kv_full + 5;  // dV, dK accumulated, dQ in TMEM        (MMA -> compute)
  uint64_t* dq_free = kv_full + 6;  // dQ read out: TMEM / tiles reusable    (compute -> MMA, 4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_full + 7);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int4 it = items[blockIdx.x];
  const MaceSeq sq = seqs[it.x];
  const int h = it.y, j = it.z;
  const int G = Hq / Hkv;
  const int W = (Hq + 2 * Hkv) * HD;
  const int n = sq.q_len;
  const int base = sq.q_start - row_offset;  // local row of token 0
  // preference-pair hole (MaceSeq): rows at or after h1 do not see keys [hole0, h1); h1 = n + 1 when there is none
  const int h1 = sq.hole_len > 0 ? sq.hole0 + sq.hole_len : n + 1;
  const int nqb = (n + 127) / 128;
  const int steps = G * (nqb - j);
  const float sl2 = scale * 1.4426950408889634f;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(&qd_full[0], 1);
    mbar_init(&qd_full[1], 1);
    mbar_init(sp_done, 1);
    mbar_init(ds_ready, 4);
    mbar_init(mm_done, 1);
    mbar_init(dq_free, 4);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  // steps: query blocks DESCENDING (outer), the GQA group's query heads (inner). Every key block's CTA reaches a
  // given (query block, head) at the same step index, so the ordered dQ accumulation (key block j waits for j - 1)
  // costs one hand-off per level instead of a lag that grows with the head index
  auto step_q = [&](int s, int& hq, int& qb) {
    hq = h * G + s % G;
    qb = nqb - 1 - s / G;
  };

  if (warp == 4) {
    // ------------------------------------------------ control warp: TMA + MMA issue (one elected lane)
    auto load_qd = [&](int s) {
      int hq, qb;
      step_q(s, hq, qb);
      uint8_t* qd = smem + C::QD_OFF + (s & 1) * 2 * C::TILE;
      mbar_arrive_expect_tx(&qd_full[s & 1], 2 * C::TILE);
#pragma unroll
      for (int a = 0; a < C::KATOMS; ++a) {
        tma_load_2d(qd + a * C::ATOM_BYTES, &maps.qkv, &qd_full[s & 1], hq * HD + a * C::ATOM, base + qb * 128);
        tma_load_2d(qd + C::TILE + a * C::ATOM_BYTES, &maps.dout, &qd_full[s & 1], hq * HD + a * C::ATOM,
                    base + qb * 128);
      }
    };
    if (elect_one()) {
      mbar_arrive_expect_tx(kv_full, 2 * C::TILE);
#pragma unroll
      for (int a = 0; a < C::KATOMS; ++a) {
        tma_load_2d(smem + C::K_OFF + a * C::ATOM_BYTES, &maps.qkv, kv_full, (Hq + h) * HD + a * C::ATOM,
                    base + j * 128);
        tma_load_2d(smem + C::V_OFF + a * C::ATOM_BYTES, &maps.qkv, kv_full, (Hq + Hkv + h) * HD + a * C::ATOM,
                    base + j * 128);
      }
      load_qd(0);
    }
    __syncwarp();
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);  // A K-major, B K-major
    constexpr uint32_t idesc_v = idesc_bf16_f32(128, HD, false, true);    // A (TMEM / K-major), B MN-major
    constexpr uint32_t idesc_q = idesc_bf16_f32(128, HD, true, true);     // A MN-major (dS), B MN-major (K)
    const uint32_t k_s = smem_u32(smem + C::K_OFF), v_s = smem_u32(smem + C::V_OFF);
    const uint32_t ds_s = smem_u32(smem + C::DS_OFF);
    mbar_wait(kv_full, 0);
    for (int s = 0; s < steps; ++s) {
      const uint32_t q_s = smem_u32(smem + C::QD_OFF + (s & 1) * 2 * C::TILE);
      const uint32_t do_s = q_s + C::TILE;
      if (s > 0) mbar_wait(dq_free, (s - 1) & 1);  // step s-1 fully consumed: TMEM S region and its tiles free
      if (s + 1 < steps) {
        if (elect_one()) load_qd(s + 1);  // buffer (s+1)&1 was last read by step s-1's MMAs
        __syncwarp();
      }
      mbar_wait(&qd_full[s & 1], (s >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const int a = (k * 16) / C::ATOM, off = ((k * 16) % C::ATOM) * 2;
          umma_bf16(tmem + C::COL_S, smem_desc(k_s + a * C::ATOM_BYTES + off, 16, 1024, 2u),
                    smem_desc(q_s + a * C::ATOM_BYTES + off, 16, 1024, 2u), idesc_s, k > 0 ? 1u : 0u);
          umma_bf16(tmem + C::COL_P, smem_desc(v_s + a * C::ATOM_BYTES + off, 16, 1024, 2u),
                    smem_desc(do_s + a * C::ATOM_BYTES + off, 16, 1024, 2u), idesc_s, k > 0 ? 1u : 0u);
        }
        umma_commit(sp_done);
      }
      __syncwarp();
      mbar_wait(ds_ready, s & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // K = 128 queries (dV, dK) / 128 keys (dQ), 16 per instruction
          const uint32_t acc = (s > 0 || k > 0) ? 1u : 0u;
          umma_bf16_ts(tmem + C::COL_DV, tmem + C::COL_P + k * 8,
                       smem_desc(do_s + k * 16 * C::SWZ, C::ATOM_BYTES, 8 * C::SWZ, 2u), idesc_v, acc);
          const int a = (k * 16) / 64, off = ((k * 16) % 64) * 2;
          umma_bf16(tmem + C::COL_DK, smem_desc(ds_s + a * 16384 + off, 16, 1024, 2u),
                    smem_desc(q_s + k * 16 * C::SWZ, C::ATOM_BYTES, 8 * C::SWZ, 2u), idesc_v, acc);
          umma_bf16(tmem + C::COL_S, smem_desc(ds_s + k * 2048, 16384, 1024, 2u),
                    smem_desc(k_s + k * 16 * C::SWZ, C::ATOM_BYTES, 8 * C::SWZ, 2u), idesc_q, k > 0 ? 1u : 0u);
        }
        umma_commit(mm_done);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ compute warps 0..3 (thread r = TMEM lane r)
    const int r = threadIdx.x;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t ds_s = smem_u32(smem + C::DS_OFF);
    float* l2_s = reinterpret_cast<float*>(smem + C::LD_OFF);
    float* d_s = l2_s + 128;
    const int kg = j * 128 + r;  // this thread's key (S^T phase)
    for (int s = 0; s < steps; ++s) {
      int hq, qb;
      step_q(s, hq, qb);
      // ---- the step's 128 query rows of lse (x log2e) and D -> smem (one load per thread instead of 128
      // dependent broadcast loads per thread); every reader of the previous step passed mm_done already
      const int q0 = qb * 128;
      {
        const int q = q0 + r;
        const bool ok = q < n;
        l2_s[r] = ok ? __ldg(lse + (size_t)(base + q) * Hq + hq) * 1.4426950408889634f : 0.f;
        d_s[r] = ok ? __ldg(Dv + (size_t)(base + q) * Hq + hq) : 0.f;
      }
      named_bar_sync(1, 128);
      mbar_wait(sp_done, s & 1);
      tc_fence_after();
      // ---- P^T, dS^T (thread = key row); P^T -> TMEM bf16, dS -> smem
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(tmem + lane_base + C::COL_S + c0, sv);
        tmem_ld_32x32b_x32(tmem + lane_base + C::COL_P + c0, dv);
        tmem_ld_wait();
        uint32_t pp[16], dd[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float p2[2], d2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int q = q0 + c0 + c + e;
            const bool ok = q < n && kg < n && kg <= q && !(q >= h1 && kg >= sq.hole0 && kg < h1);
            const float p = ok ? exp2f(__uint_as_float(sv[c + e]) * sl2 - l2_s[c0 + c + e]) : 0.f;
            p2[e] = p;
            d2[e] = p * (__uint_as_float(dv[c + e]) - d_s[c0 + c + e]);
          }
          pp[c / 2] = pack_bf16(p2[0], p2[1]);
          dd[c / 2] = pack_bf16(d2[0], d2[1]);
        }
        // P^T columns [c0/2, c0/2 + 16) of the P region: dP^T columns already pulled into registers
        tmem_st_32x32b_x16(tmem + lane_base + C::COL_P + c0 / 2, pp);
        // dS row r (key), queries c0..c0+31: 4 16-byte chunks of the swizzled [128 keys][128 queries] tile
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const int qc = c0 + ch * 8;  // first query of the chunk
          const int atom = qc / 64, chunk = (qc % 64) / 8;
          st_shared_v4(ds_s + atom * 16384 + r * 128 + ((chunk ^ (r & 7)) << 4), dd[ch * 4], dd[ch * 4 + 1],
                       dd[ch * 4 + 2], dd[ch * 4 + 3]);
        }
      }
      tmem_st_wait();
      fence_proxy_async_shared();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_ready);
      mbar_wait(mm_done, s & 1);
      tc_fence_after();
      // ---- dQ rows (thread = query row). Key blocks j = 0..qb contribute to query block qb: with dq_order the
      // contributions are added in ascending j (a per-(query block, head) counter: wait for j, add, publish j + 1;
      // the last contributor resets it), so dQ is bitwise reproducible; without it, fp32 atomics
      const int qg = q0 + r;
      float* dq_row = dqkv + (size_t)(base + qg) * W + hq * HD;
      int* ctr = dq_order ? dq_order + (size_t)(base + q0) * Hq + hq : nullptr;
      if (ctr) {
        if (r == 0) order_wait(ctr, j);
        named_bar_sync(1, 128);
      }
#pragma unroll 1
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + lane_base + C::COL_S + c0, v);
        tmem_ld_wait();
        if (qg < n) {
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            if (ctr) {
              float4* p4 = reinterpret_cast<float4*>(dq_row + c0 + c);
              float4 x = __ldcg(p4);
              x.x += __uint_as_float(v[c]) * scale;
              x.y += __uint_as_float(v[c + 1]) * scale;
              x.z += __uint_as_float(v[c + 2]) * scale;
              x.w += __uint_as_float(v[c + 3]) * scale;
              __stcg(p4, x);
            } else {
              red_add_v4(dq_row + c0 + c, __uint_as_float(v[c]) * scale, __uint_as_float(v[c + 1]) * scale,
                         __uint_as_float(v[c + 2]) * scale, __uint_as_float(v[c + 3]) * scale);
            }
          }
        }
      }
      if (ctr) {
        __threadfence();
        named_bar_sync(1, 128);
        if (r == 0) order_release(ctr, j == qb ? 0 : j + 1);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_free);
    }
    // ---- dK (x scale), dV rows of this key block (thread = key row; exclusive owner)
    tc_fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < HD; c0 += 32) {  // tcgen05.ld is warp-collective: rows past n load and drop
      uint32_t a[32], b[32];
      tmem_ld_32x32b_x32(tmem + lane_base + C::COL_DK + c0, a);
      tmem_ld_32x32b_x32(tmem + lane_base + C::COL_DV + c0, b);
      tmem_ld_wait();
      if (kg < n) {
        float* dk_row = dqkv + (size_t)(base + kg) * W + (Hq + h) * HD;
        float* dv_row = dqkv + (size_t)(base + kg) * W + (Hq + Hkv + h) * HD;
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          *reinterpret_cast<float4*>(dk_row + c0 + c) =
              make_float4(__uint_as_float(a[c]) * scale, __uint_as_float(a[c + 1]) * scale,
                          __uint_as_float(a[c + 2]) * scale, __uint_as_float(a[c + 3]) * scale);
          *reinterpret_cast<float4*>(dv_row + c0 + c) =
              make_float4(__uint_as_float(b[c]), __uint_as_float(b[c + 1]), __uint_as_float(b[c + 2]),
                          __uint_as_float(b[c + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

static bool bwd_map(MaceCtx* ctx, CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows) {
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  return ctx->encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD>
static int launch_bwd_tc(MaceCtx* ctx, const void* qkv, const void* dout, const float* lse, int n_rows, int Hq, int Hkv,
                         const MaceSeq* seqs, const int* items, int n_items, int row_offset, const float* Dbuf,
                         float* dqkv, int* dq_order, cudaStream_t s) {
  using C = BwdCfg<HD>;
  BwdMaps maps;
  const int W = (Hq + 2 * Hkv) * HD;
  if (!bwd_map(ctx, &maps.qkv, qkv, W, n_rows) || !bwd_map(ctx, &maps.dout, dout, (uint64_t)Hq * HD, n_rows))
    return mace_fail(ctx, MACE_ERR_LAUNCH, "attn_bwd: tensor map encode failed");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_bwd_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  launch_k(attn_bwd_tc_kernel<HD>, n_items, 160, C::SMEM, s, maps, lse, Dbuf, seqs,
           reinterpret_cast<const int4*>(items), Hq, Hkv, 1.f / sqrtf((float)HD), dqkv, row_offset, dq_order);
  ctx->launches++;
  return 0;
}

int attn_bwd_tc(MaceCtx* ctx, const void* qkv, const void* dout, const float* lse, int n_rows, int Hq, int Hkv, int hd,
                const MaceSeq* seqs, const int* items, int n_items, int row_offset, const float* Dbuf, float* dqkv,
                int* dq_order, cudaStream_t s) {
  if (hd == 64)
    return launch_bwd_tc<64>(ctx, qkv, dout, lse, n_rows, Hq, Hkv, seqs, items, n_items, row_offset, Dbuf, dqkv,
                             dq_order, s);
  return launch_bwd_tc<128>(ctx, qkv, dout, lse, n_rows, Hq, Hkv, seqs, items, n_items, row_offset, Dbuf, dqkv,
                            dq_order, s);
}

}  // namespace mace
