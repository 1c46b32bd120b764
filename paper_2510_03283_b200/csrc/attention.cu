// Ragged paged attention forward for the hybrid iteration: prefill, decode and fine-tune sequences of
// one tick in one call (reference stand-ins replaced: Engine._exec_prefill engine.py:444-480,
// Engine._exec_decode engine.py:482-532, the FT pair forward behind AlignmentEnv.pair_loss
// alignment.py:151-166).
//
//  * tc path (prefill + fine-tune sequences, tensor-core bound): CTA = 128 query rows x 1 query head.
//    Q tile and K/V tiles of 128 tokens (8 pages of 16) are TMA-staged with hardware swizzle,
//    S = Q.K^T and P.V run as tcgen05.mma with fp32 accumulators in TMEM; thread i owns query row i
//    (TMEM lane i) for the online softmax; the P.V partial is folded into registers so the next S tile
//    overlaps the accumulation. Paged K/V come from the head-major page pools, dense FT K/V straight
//    from the packed qkv rows.
//  * decode path (HBM bound): attention_decode.cu (warp per (sequence, kv head, chunk) item).
#include <cmath>

#include "common.cuh"
#include "mace_internal.h"

namespace mace {

constexpr float kLog2e = 1.4426950408889634f;

// =====================================================================================================
// tensor-core path
// =====================================================================================================
template <int HD>
struct TcCfg {
  static constexpr int SWZ = HD >= 64 ? 128 : 64;     // bytes per swizzled row
  static constexpr int ATOM = SWZ / 2;                // bf16 elements per swizzle row
  static constexpr int KATOMS = HD / ATOM;            // swizzle atoms along head_dim
  static constexpr uint32_t LAYOUT = SWZ == 128 ? 2u : 4u;
  static constexpr int TILE = 128 * HD * 2;           // one 128-row Q/K/V tile
  static constexpr int ATOM_BYTES = 128 * SWZ;        // one 128-row atom column block
  static constexpr int P_BYTES = 128 * 128 * 2;
  static constexpr int Q_OFF = 0;
  static constexpr int KV_OFF = TILE;                 // stage s: K at KV_OFF + 2s*TILE, V at +TILE
  static constexpr int P_OFF = 5 * TILE;
  static constexpr int BAR_OFF = P_OFF + P_BYTES;
  static constexpr int NEED = BAR_OFF + 128;
  // keep <= 2 CTAs per SM so two 256-column TMEM allocations always fit
  static constexpr int SMEM = (NEED + 1024) < 80 * 1024 ? 80 * 1024 : (NEED + 1024);
};

struct TcMaps {
  CUtensorMap q;       // qkv [T, W], box {ATOM, 128}
  CUtensorMap dense;   // qkv [T, W], box {ATOM, 16}
  CUtensorMap kpool;   // [pages*16, HD], box {ATOM, 16}
  CUtensorMap vpool;
};

template <int HD>
__global__ void __launch_bounds__(128) attn_tc_kernel(const __grid_constant__ TcMaps maps, const MaceSeq* __restrict__ seqs,
                                                      const int4* __restrict__ items, const MaceKvLayout kv, int Hq,
                                                      int Hkv, float scale_log2, __nv_bfloat16* __restrict__ out,
                                                      float* __restrict__ lse_out) {
  using C = TcCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar_q = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* bar_full = bar_q + 1;  // [2]
  uint64_t* bar_s = bar_q + 3;
  uint64_t* bar_o = bar_q + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_q + 5);

  const int4 it = items[blockIdx.x];
  const MaceSeq sq = seqs[it.x];
  const int hq = it.y, qb = it.z;
  const int h = hq / (Hq / Hkv);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int W = (Hq + 2 * Hkv) * HD;
  const bool dense = sq.kind == 2;
  const int kv_len = sq.kv_len;
  const int q0 = qb * 128;
  const int q_last_log = kv_len - sq.q_len + min(q0 + 127, sq.q_len - 1);  // causal horizon of the tile
  const int n_tiles = q_last_log / 128 + 1;

  if (tid == 0) {
    mbar_init(bar_q, 1);
    mbar_init(&bar_full[0], 1);
    mbar_init(&bar_full[1], 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();
  const uint32_t tmem_s = tmem, tmem_o = tmem + 128;

  auto load_kv = [&](int j, int stage) {
    uint8_t* ks = smem + C::KV_OFF + 2 * stage * C::TILE;
    uint8_t* vs = ks + C::TILE;
    mbar_arrive_expect_tx(&bar_full[stage], 2 * C::TILE);
#pragma unroll 1
    for (int pslot = 0; pslot < 8; ++pslot) {
      const int tok0 = j * 128 + pslot * 16;
      if (dense) {
        const int row = sq.q_start + tok0;  // FT: kv rows = q rows
#pragma unroll
        for (int a = 0; a < C::KATOMS; ++a) {
          tma_load_2d(ks + a * C::ATOM_BYTES + pslot * 16 * C::SWZ, &maps.dense, &bar_full[stage],
                      (Hq + h) * HD + a * C::ATOM, row);
          tma_load_2d(vs + a * C::ATOM_BYTES + pslot * 16 * C::SWZ, &maps.dense, &bar_full[stage],
                      (Hq + Hkv + h) * HD + a * C::ATOM, row);
        }
      } else {
        int lp = tok0 / 16;
        const int maxp = (kv_len + 15) / 16;
        if (lp >= maxp) lp = maxp - 1;  // beyond the sequence: any valid page, masked below
        const int page = kv.ptab[(size_t)sq.slot * kv.max_prompt_pages + lp] * Hkv + h;
#pragma unroll
        for (int a = 0; a < C::KATOMS; ++a) {
          tma_load_2d(ks + a * C::ATOM_BYTES + pslot * 16 * C::SWZ, &maps.kpool, &bar_full[stage], a * C::ATOM,
                      page * 16);
          tma_load_2d(vs + a * C::ATOM_BYTES + pslot * 16 * C::SWZ, &maps.vpool, &bar_full[stage], a * C::ATOM,
                      page * 16);
        }
      }
    }
  };

  constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);
  constexpr uint32_t idesc_o = idesc_bf16_f32(128, HD, false, true);
  auto issue_s = [&](int stage) {
    const uint32_t qa = smem_u32(smem + C::Q_OFF);
    const uint32_t ka = smem_u32(smem + C::KV_OFF + 2 * stage * C::TILE);
#pragma unroll
    for (int k = 0; k < HD / 16; ++k) {
      const int a = (k * 16) / C::ATOM, off = ((k * 16) % C::ATOM) * 2;
      const uint64_t ad = smem_desc(qa + a * C::ATOM_BYTES + off, 16, 8 * C::SWZ, C::LAYOUT);
      const uint64_t bd = smem_desc(ka + a * C::ATOM_BYTES + off, 16, 8 * C::SWZ, C::LAYOUT);
      umma_bf16(tmem_s, ad, bd, idesc_s, k > 0 ? 1u : 0u);
    }
    umma_commit(bar_s);
  };
  auto issue_o = [&](int stage) {
    const uint32_t pa = smem_u32(smem + C::P_OFF);
    const uint32_t va = smem_u32(smem + C::KV_OFF + 2 * stage * C::TILE + C::TILE);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t ad = smem_desc(pa + (k / 4) * 16384 + (k % 4) * 32, 16, 1024, 2u);
      const uint64_t bd = smem_desc(va + k * 16 * C::SWZ, C::ATOM_BYTES, 8 * C::SWZ, C::LAYOUT);
      umma_bf16(tmem_o, ad, bd, idesc_o, k > 0 ? 1u : 0u);
    }
    umma_commit(bar_o);
  };

  if (tid == 0) {
    mbar_arrive_expect_tx(bar_q, C::TILE);
#pragma unroll
    for (int a = 0; a < C::KATOMS; ++a)
      tma_load_2d(smem + C::Q_OFF + a * C::ATOM_BYTES, &maps.q, bar_q, hq * HD + a * C::ATOM, sq.q_start + q0);
    load_kv(0, 0);
    if (n_tiles > 1) load_kv(1, 1);
    mbar_wait(bar_q, 0);
    mbar_wait(&bar_full[0], 0);
    tc_fence_after();
    issue_s(0);
  }

  const int qi = q0 + tid;                         // query row within the sequence
  const bool q_ok = qi < sq.q_len;
  const int q_log = kv_len - sq.q_len + qi;        // its logical kv index (causal horizon)
  float m_run = -INFINITY, l_run = 0.f;
  float o_acc[HD];
#pragma unroll
  for (int d = 0; d < HD; ++d) o_acc[d] = 0.f;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  uint8_t* p_row = smem + C::P_OFF + tid * 128;

  for (int j = 0; j < n_tiles; ++j) {
    mbar_wait(bar_s, j & 1);
    tc_fence_after();
    // ---- pass 1: row max over the valid, causal columns
    const int lim = min(kv_len - 1, q_log) - j * 128;  // last valid column in this tile
    float mx = -INFINITY;
#pragma unroll 1
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_s + lane_base + c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c0 + c <= lim) mx = fmaxf(mx, __uint_as_float(r[c]));
    }
    const float m_new = fmaxf(m_run, mx * scale_log2);
    const float alpha = (m_run == -INFINITY) ? 0.f : exp2f(m_run - m_new);
    // ---- pass 2: P = exp2(s*scale - m) -> bf16 into the swizzled K-major A tile
    float psum = 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem_s + lane_base + c0, r);
      tmem_ld_wait();
      float p[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        p[c] = (c0 + c <= lim && m_new != -INFINITY) ? exp2f(__uint_as_float(r[c]) * scale_log2 - m_new) : 0.f;
        psum += p[c];
      }
      const int atom = c0 / 64;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const int chunk = ((c0 % 64) / 8) + ch;  // 16-byte chunk within the 128-byte row
        uint4 v = make_uint4(pack_bf16(p[ch * 8], p[ch * 8 + 1]), pack_bf16(p[ch * 8 + 2], p[ch * 8 + 3]),
                             pack_bf16(p[ch * 8 + 4], p[ch * 8 + 5]), pack_bf16(p[ch * 8 + 6], p[ch * 8 + 7]));
        *reinterpret_cast<uint4*>(p_row + atom * 16384 + ((chunk ^ (tid & 7)) * 16)) = v;
      }
    }
    l_run = l_run * alpha + psum;
    m_run = m_new;
    tc_fence_before();
    fence_proxy_async_shared();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      issue_o(j & 1);
      if (j + 1 < n_tiles) {
        mbar_wait(&bar_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
        tc_fence_after();
        issue_s((j + 1) & 1);
      }
    }
    mbar_wait(bar_o, j & 1);
    tc_fence_after();
#pragma unroll
    for (int c0 = 0; c0 < HD; c0 += 16) {
      uint32_t r[16];
      tmem_ld_32x32b_x16(tmem_o + lane_base + c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 16; ++c) o_acc[c0 + c] = o_acc[c0 + c] * alpha + __uint_as_float(r[c]);
    }
    if (tid == 0 && j + 2 < n_tiles) load_kv(j + 2, j & 1);
  }

  if (q_ok) {
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    const int row = sq.q_start + qi;
    __nv_bfloat16* o = out + (size_t)row * Hq * HD + hq * HD;
#pragma unroll
    for (int d = 0; d < HD; d += 8) {
      uint4 v = make_uint4(pack_bf16(o_acc[d] * inv, o_acc[d + 1] * inv), pack_bf16(o_acc[d + 2] * inv, o_acc[d + 3] * inv),
                           pack_bf16(o_acc[d + 4] * inv, o_acc[d + 5] * inv), pack_bf16(o_acc[d + 6] * inv, o_acc[d + 7] * inv));
      *reinterpret_cast<uint4*>(o + d) = v;
    }
    if (lse_out) lse_out[(size_t)row * Hq + hq] = (m_run + log2f(l_run)) / kLog2e;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
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
  using C = TcCfg<HD>;
  TcMaps maps;
  const int W = (a->Hq + 2 * a->Hkv) * HD;
  bool ok = encode_2d(ctx, &maps.q, a->qkv, W, a->T, W, C::ATOM, 128, C::SWZ) &&
            encode_2d(ctx, &maps.dense, a->qkv, W, a->T, W, C::ATOM, 16, C::SWZ);
  const void* kp = a->k_pool ? a->k_pool : a->qkv;
  const void* vp = a->v_pool ? a->v_pool : a->qkv;
  const uint64_t rows = a->k_pool ? (uint64_t)a->pool_pages * 16 : (uint64_t)a->T;
  const uint64_t ld = a->k_pool ? HD : W;
  ok = ok && encode_2d(ctx, &maps.kpool, kp, HD, rows, ld, C::ATOM, 16, C::SWZ) &&
       encode_2d(ctx, &maps.vpool, vp, HD, rows, ld, C::ATOM, 16, C::SWZ);
  if (!ok) return mace_fail(ctx, MACE_ERR_LAUNCH, "attn: tensor map encode failed");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  launch_k(attn_tc_kernel<HD>, a->n_tc, 128, C::SMEM, s, maps, a->seqs, reinterpret_cast<const int4*>(a->tc_items), a->kv,
                                                   a->Hq, a->Hkv, scale_log2, (__nv_bfloat16*)a->out, a->lse);
  ctx->launches++;
  return 0;
}

int dispatch_decode2(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s);
int dispatch_decode_tc(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s);

}  // namespace mace

using namespace mace;

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
