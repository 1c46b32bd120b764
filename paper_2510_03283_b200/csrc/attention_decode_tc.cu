// Paged decode attention on the tensor cores (tcgen05, "swap-AB"): the B200-native form of the
// HBM-bound decode hot kernel (reference stand-in: Engine._exec_decode, engine.py:482-532).
//
// A decode row has 1 query per query head; its GQA group (G heads, padded to N=16) is the MMA's N
// dimension and the KV tokens are M, so S^T = K . Q^T puts one TOKEN per TMEM lane:
//   * per item (decode sequence, kv head, chunk of its page list) a CTA streams 128-token tiles =
//     8 head-major pages, K and V each fetched by one 2-D TMA box per page (128B swizzle), through a
//     STAGES-deep mbarrier ring;
//   * S^T[128 tok, 16] = K[128, hd] . Q^T  (tcgen05.mma M=128 N=16, fp32 in TMEM);
//   * thread t = token t: tcgen05.ld its 16 scores, masks the page's invalid rows (per-head decode
//     window, prompt tail), online softmax per head (one CTA reduction for the max; per-warp sums),
//     writes P^T (bf16, K-major swizzled) for the next MMA;
//   * O^T[hd, 16] += V^T[hd, 128 tok] . P  (tcgen05.mma, A = V pages read MN-major), accumulated in
//     registers by thread r = head dim r; the S MMA of the next tile is issued before the P.V result is
//     consumed so the tensor core overlaps the softmax.
// The CUDA cores only do the softmax, so G query heads per KV byte (GQA) cost no extra SM time.
// Multi-chunk items write (m, l, o) partials merged in chunk order by the last CTA (deterministic).
#include <cmath>

#include "common.cuh"
#include "mace_internal.h"

namespace mace {

template <int HD>
struct DecTc {
  static constexpr int SWZ = HD >= 64 ? 128 : 64;
  static constexpr int ATOM = SWZ / 2;
  static constexpr int KATOMS = HD / ATOM;
  static constexpr uint32_t LAYOUT = SWZ == 128 ? 2u : 4u;
  static constexpr int ATOM_BYTES = 128 * SWZ;          // 128 token rows x one swizzle atom of head dims
  static constexpr int TILE = KATOMS * ATOM_BYTES;      // one K (or V) tile of 128 tokens
  static constexpr int STAGES = HD >= 128 ? 2 : 3;
  static constexpr int KV_OFF = 0;                      // stage s: K at 2s*TILE, V at (2s+1)*TILE
  static constexpr int Q_OFF = STAGES * 2 * TILE;       // [16 rows][HD] K-major, KATOMS atoms of 16*SWZ
  static constexpr int Q_BYTES = KATOMS * 16 * SWZ;
  static constexpr int P_OFF = Q_OFF + Q_BYTES;         // P^T [16 rows][128 tok] K-major SW128 (2 atoms)
  static constexpr int P_BYTES = 2 * 16 * 128;
  static constexpr int RED_OFF = P_OFF + P_BYTES;       // float [4 warps][16] + [4][16]
  static constexpr int BAR_OFF = RED_OFF + 2 * 4 * 16 * 4;
  static constexpr int SMEM = BAR_OFF + 128 + 1024;
  static constexpr int PARTIAL(int G) { return 2 * G + G * HD; }
};

template <int HD, int G>
__global__ void __launch_bounds__(128) attn_decode_tc_kernel(
    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
    const __nv_bfloat16* __restrict__ qkv, const MaceSeq* __restrict__ seqs, const int4* __restrict__ items,
    const MaceKvLayout kv, int Hq, int Hkv, float scale_log2, __nv_bfloat16* __restrict__ out,
    float* __restrict__ head_norm, float* __restrict__ partials, int* __restrict__ counters) {
  using C = DecTc<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* red_max = reinterpret_cast<float*>(smem + C::RED_OFF);
  float* red_sum = red_max + 4 * 16;
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);  // [STAGES]
  uint64_t* bar_s = bar_full + C::STAGES;
  uint64_t* bar_o = bar_s + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_o + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- zero the V stages, Q and P once: skipped page slots and padded heads must multiply as finite
  // zeros (K rows of skipped slots are masked by index, never by value)
  for (int s = 0; s < C::STAGES; ++s)
    for (int i = tid * 16; i < C::TILE; i += 128 * 16)
      *reinterpret_cast<uint4*>(smem + C::KV_OFF + (2 * s + 1) * C::TILE + i) = make_uint4(0, 0, 0, 0);
  for (int i = C::Q_OFF + tid * 16; i < C::P_OFF + C::P_BYTES; i += 128 * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&bar_full[s], 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<32>(tmem_slot);
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_s = tmem, tmem_o = tmem + 16;
  pdl_wait();
  pdl_trigger();

  const int4 it = items[blockIdx.x];
  const MaceSeq sq = seqs[it.x];
  const int h = it.y, chunk = it.z >> 16, nch = it.z & 0xffff;
  const int W = (Hq + 2 * Hkv) * HD;
  // ---- Q rows (G query heads of the group) -> K-major swizzled B operand, rows >= G stay zero
  {
    const __nv_bfloat16* qrow = qkv + (size_t)sq.q_start * W + (size_t)h * G * HD;
    for (int i = tid; i < G * (HD / 8); i += 128) {
      const int g = i / (HD / 8), c = i % (HD / 8);  // 16-byte chunk c of head g
      const int a = (c * 8) / C::ATOM, cc = c % (C::SWZ / 16);
      const int sw = C::SWZ == 128 ? (cc ^ (g & 7)) : (cc ^ ((g >> 1) & 3));
      *reinterpret_cast<uint4*>(smem + C::Q_OFF + a * 16 * C::SWZ + g * C::SWZ + sw * 16) =
          *reinterpret_cast<const uint4*>(qrow + g * HD + c * 8);
    }
    fence_proxy_async_shared();  // generic-proxy Q writes -> visible to the tensor core
    __syncthreads();
  }
  // ---- this chunk's page slots (same split as the CUDA-core path)
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
  const int n_tiles = (n_pg + 7) / 8;
  auto slot_info = [&](int p, int& page, int& lo, int& hi) {  // p = page slot within the chunk
    const int ps = s0 + p;
    if (ps >= s1) {
      page = -1;
      lo = hi = 0;
    } else if (ps < npp) {
      page = kv.ptab[(size_t)sq.slot * kv.max_prompt_pages + ps] * Hkv + h;
      lo = 0;
      hi = min(16, n_pv - 16 * ps);
    } else {
      const int r = r0 + (ps - npp);
      page = kv.dtab[(size_t)kvh * kv.max_dec_pages + r];
      const int b = db + 16 * r;
      lo = max(0, d0 - b);
      hi = min(16, de - b);
    }
  };
  auto load_tile = [&](int j, int st) {
    uint8_t* ks = smem + C::KV_OFF + 2 * st * C::TILE;
    uint8_t* vs = ks + C::TILE;
    int nbox = 0;
    int pages[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int lo, hi;
      slot_info(8 * j + q, pages[q], lo, hi);
      nbox += pages[q] >= 0;
    }
    mbar_arrive_expect_tx(&bar_full[st], nbox * 2 * C::KATOMS * 16 * C::SWZ);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (pages[q] < 0) continue;
#pragma unroll
      for (int a = 0; a < C::KATOMS; ++a) {
        tma_load_2d(ks + a * C::ATOM_BYTES + q * 16 * C::SWZ, &kmap, &bar_full[st], a * C::ATOM, pages[q] * 16);
        tma_load_2d(vs + a * C::ATOM_BYTES + q * 16 * C::SWZ, &vmap, &bar_full[st], a * C::ATOM, pages[q] * 16);
      }
    }
  };
  constexpr uint32_t idesc_s = idesc_bf16_f32(128, 16, false, false);
  constexpr uint32_t idesc_o = idesc_bf16_f32(128, 16, true, false);
  auto issue_s = [&](int st) {
    const uint32_t ka = smem_u32(smem + C::KV_OFF + 2 * st * C::TILE);
    const uint32_t qa = smem_u32(smem + C::Q_OFF);
#pragma unroll
    for (int k = 0; k < HD / 16; ++k) {
      const int a = (k * 16) / C::ATOM, off = ((k * 16) % C::ATOM) * 2;
      const uint64_t ad = smem_desc(ka + a * C::ATOM_BYTES + off, 16, 8 * C::SWZ, C::LAYOUT);
      const uint64_t bd = smem_desc(qa + a * 16 * C::SWZ + off, 16, 8 * C::SWZ, C::LAYOUT);
      umma_bf16(tmem_s, ad, bd, idesc_s, k > 0 ? 1u : 0u);
    }
    umma_commit(bar_s);
  };
  auto issue_o = [&](int st) {
    const uint32_t va = smem_u32(smem + C::KV_OFF + (2 * st + 1) * C::TILE);
    const uint32_t pa = smem_u32(smem + C::P_OFF);
    // A = V^T (M = head dims, MN-major; M=128 pads head dims by re-reading the same atom: LBO 0 for a
    // single 64-wide atom), B = P^T (N = 16 heads, K-major over 128 tokens)
    constexpr uint32_t lbo = C::KATOMS > 1 ? C::ATOM_BYTES : 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t ad = smem_desc(va + k * 16 * C::SWZ, lbo, 8 * C::SWZ, C::LAYOUT);
      const uint64_t bd = smem_desc(pa + (k / 4) * (16 * 128) + (k % 4) * 32, 16, 1024, 2u);
      umma_bf16(tmem_o, ad, bd, idesc_o, k > 0 ? 1u : 0u);
    }
    umma_commit(bar_o);
  };

  if (tid == 0 && n_tiles > 0) {
    for (int j = 0; j < n_tiles && j < C::STAGES; ++j) load_tile(j, j);
    mbar_wait(&bar_full[0], 0);
    tc_fence_after();
    issue_s(0);
  }

  float m_run[G], l_warp[G], o_acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m_run[g] = -INFINITY;
    l_warp[g] = 0.f;
    o_acc[g] = 0.f;
  }
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const int q = tid >> 4, row = tid & 15;  // this thread's token: page slot q, row in page
  for (int j = 0; j < n_tiles; ++j) {
    const int st = j % C::STAGES;
    int pg, lo, hi;
    slot_info(8 * j + q, pg, lo, hi);
    const bool valid = pg >= 0 && row >= lo && row < hi;
    mbar_wait(bar_s, j & 1);
    tc_fence_after();
    uint32_t sr[16];
    tmem_ld_32x32b_x16(tmem_s + lane_base, sr);
    tmem_ld_wait();
    // ---- tile max per head: warp max, then across the 4 warps
    float sv[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      sv[g] = valid ? __uint_as_float(sr[g]) * scale_log2 : -INFINITY;
      const float mx = warp_max(sv[g]);
      if (lane == 0) red_max[warp * 16 + g] = mx;
    }
    __syncthreads();
    float alpha[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float mt = fmaxf(fmaxf(red_max[g], red_max[16 + g]), fmaxf(red_max[32 + g], red_max[48 + g]));
      const float mn = fmaxf(m_run[g], mt);
      alpha[g] = (m_run[g] == -INFINITY) ? (mn == -INFINITY ? 1.f : 0.f) : exp2f(m_run[g] - mn);
      m_run[g] = mn;
      const float p = valid ? exp2f(sv[g] - mn) : 0.f;
      l_warp[g] = l_warp[g] * alpha[g] + warp_sum(p);
      // P^T[g][tid]: K-major SW128, atom tid/64, 16-byte chunk (tid%64)/8 swizzled by row g
      const int ch = ((tid & 63) >> 3) ^ (g & 7);
      *reinterpret_cast<__nv_bfloat16*>(smem + C::P_OFF + (tid >> 6) * (16 * 128) + g * 128 + ch * 16 + (tid & 7) * 2) =
          __float2bfloat16(p);
    }
    tc_fence_before();
    fence_proxy_async_shared();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      issue_o(st);
      if (j + 1 < n_tiles) {
        const int st1 = (j + 1) % C::STAGES;
        mbar_wait(&bar_full[st1], ((j + 1) / C::STAGES) & 1);
        tc_fence_after();
        issue_s(st1);
      }
    }
    mbar_wait(bar_o, j & 1);
    tc_fence_after();
    uint32_t orr[16];
    tmem_ld_32x32b_x16(tmem_o + lane_base, orr);  // thread r <-> head dim r (rows >= HD are padding)
    tmem_ld_wait();
#pragma unroll
    for (int g = 0; g < G; ++g) o_acc[g] = o_acc[g] * alpha[g] + __uint_as_float(orr[g]);
    tc_fence_before();
    __syncthreads();  // stage st fully consumed (S of tile j and P.V of tile j completed)
    if (tid == 0 && j + C::STAGES < n_tiles) load_tile(j + C::STAGES, st);
  }

  // ---- row sums across warps, then output / partial
#pragma unroll
  for (int g = 0; g < G; ++g)
    if (lane == 0) red_sum[warp * 16 + g] = l_warp[g];
  __syncthreads();
  float l_tot[G];
#pragma unroll
  for (int g = 0; g < G; ++g) l_tot[g] = (red_sum[g] + red_sum[16 + g]) + (red_sum[32 + g] + red_sum[48 + g]);
  const int orow = sq.q_start;
  const int r = tid;  // head dim owned by this thread (< HD)
  auto emit = [&](const float* m_, const float* l_, const float* o_) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float inv = l_[g] > 0.f ? 1.f / l_[g] : 0.f;
      const float v = o_[g] * inv;
      if (r < HD) out[(size_t)orow * Hq * HD + (size_t)(h * G + g) * HD + r] = __float2bfloat16(v);
      if (head_norm) {
        float sq2 = warp_sum(r < HD ? v * v : 0.f);
        if (lane == 0) red_max[warp * 16 + g] = sq2;
      }
    }
    if (head_norm) {
      __syncthreads();
      if (tid < G)
        head_norm[(size_t)orow * Hq + h * G + tid] =
            sqrtf((red_max[tid] + red_max[16 + tid]) + (red_max[32 + tid] + red_max[48 + tid]));
    }
  };
  if (nch == 1) {
    emit(m_run, l_tot, o_acc);
  } else {
    float* mine = partials + (size_t)(it.w + chunk) * C::PARTIAL(G);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (tid == 0) {
        mine[g] = m_run[g];
        mine[G + g] = l_tot[g];
      }
      if (r < HD) mine[2 * G + g * HD + r] = o_acc[g];
    }
    __threadfence();
    __syncthreads();
    __shared__ int prev;
    if (tid == 0) prev = atomicAdd(&counters[kvh], 1);
    __syncthreads();
    if (prev == nch - 1) {
      __threadfence();
      const float* first = partials + (size_t)it.w * C::PARTIAL(G);
      float M[G], L[G], A[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        M[g] = -INFINITY;
        for (int c = 0; c < nch; ++c) M[g] = fmaxf(M[g], __ldcg(first + c * C::PARTIAL(G) + g));
        L[g] = 0.f;
        A[g] = 0.f;
        for (int c = 0; c < nch; ++c) {  // chunk order: deterministic
          const float* pc = first + c * C::PARTIAL(G);
          const float mc = __ldcg(pc + g);
          const float sc = mc == -INFINITY ? 0.f : exp2f(mc - M[g]);
          L[g] += __ldcg(pc + G + g) * sc;
          if (r < HD) A[g] += __ldcg(pc + 2 * G + g * HD + r) * sc;
        }
      }
      emit(M, L, A);
      if (tid == 0) counters[kvh] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
  }
}

static bool encode_pool(MaceCtx* ctx, CUtensorMap* m, const void* pool, long long pages, int HD, int atom, int swz) {
  cuuint64_t dims[2] = {(cuuint64_t)HD, (cuuint64_t)pages * 16};
  cuuint64_t strides[1] = {(cuuint64_t)HD * 2};
  cuuint32_t box[2] = {(cuuint32_t)atom, 16};
  cuuint32_t estr[2] = {1, 1};
  return ctx->encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD, int G>
int launch_decode_tc(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s) {
  using C = DecTc<HD>;
  CUtensorMap km, vm;
  if (!encode_pool(ctx, &km, a->k_pool, a->pool_pages, HD, C::ATOM, C::SWZ) ||
      !encode_pool(ctx, &vm, a->v_pool, a->pool_pages, HD, C::ATOM, C::SWZ))
    return mace_fail(ctx, MACE_ERR_LAUNCH, "attn decode tc: tensor map encode failed");
  const size_t need = (size_t)a->n_dec * C::PARTIAL(G) * 4;
  if (!a->dec_workspace || a->dec_workspace_bytes < need || !a->dec_counters)
    return mace_fail(ctx, MACE_ERR_ARG, "attn decode: workspace/counters too small");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_tc_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  launch_k(attn_decode_tc_kernel<HD, G>, a->n_dec, 128, C::SMEM, s, km, vm, (const __nv_bfloat16*)a->qkv, a->seqs,
           reinterpret_cast<const int4*>(a->dec_items), a->kv, a->Hq, a->Hkv, sl2, (__nv_bfloat16*)a->out,
           a->head_norm, (float*)a->dec_workspace, a->dec_counters);
  ctx->launches++;
  return 0;
}

int dispatch_decode_tc(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s) {
  const int G = a->Hq / a->Hkv;
#define MACE_DTC(HD_)                                                 \
  switch (G) {                                                        \
    case 1: return launch_decode_tc<HD_, 1>(ctx, a, sl2, s);          \
    case 2: return launch_decode_tc<HD_, 2>(ctx, a, sl2, s);          \
    case 4: return launch_decode_tc<HD_, 4>(ctx, a, sl2, s);          \
    case 8: return launch_decode_tc<HD_, 8>(ctx, a, sl2, s);          \
    default: return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn decode: GQA group must be 1, 2, 4 or 8"); \
  }
  switch (a->hd) {
    case 32: MACE_DTC(32)
    case 64: MACE_DTC(64)
    case 128: MACE_DTC(128)
    default: return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn decode: head_dim must be 32, 64 or 128");
  }
#undef MACE_DTC
}

}  // namespace mace
