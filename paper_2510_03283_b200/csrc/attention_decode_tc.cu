// Paged decode attention on the tensor cores (tcgen05, "swap-AB"), persistent and warp-specialised:
// the B200-native form of the HBM-bound decode hot kernel (reference stand-in: Engine._exec_decode,
// engine.py:482-532, with the per-head windows of the prune trim, engine.py:506-511).
//
// A decode row has 1 query per query head; its GQA group (G heads, padded to N = 16) is the MMA's N
// dimension and the KV tokens are M, so S^T = K . Q^T puts one TOKEN per TMEM lane. Work item =
// (decode sequence, kv head, chunk of its page list); items are pre-sorted longest first and dealt to
// the persistent CTAs cyclically. Roles:
//   warp 4  producer   TMA: per item the G query rows (one 2-D box), per 128-token tile 8 head-major
//                      K pages + 8 V pages (one box each), through a STAGES-deep mbarrier ring that
//                      runs across item boundaries
//   warp 5  MMA        single thread: S^T[128 tok, 16] = K . Q^T into TMEM S[t&1]; then the previous
//                      tile's O^T[hd, 16] = V^T . P (V read MN-major) into TMEM O[(t-1)&1]; commits
//                      release K/V stages, S/P/O buffers and Q buffers
//   warps 0-3 softmax  thread t = token t of the tile: masks the page's invalid rows, online softmax per
//                      head (one cross-warp max per tile), P^T (bf16, K-major swizzled) to smem; thread
//                      r = head dim r folds each tile's P.V result into registers; epilogue / chunk merge
// Double-buffered S, P and O let the tensor core run tile t+1's S and tile t's P.V while the CUDA
// cores do tile t's softmax. Multi-chunk items write (m, l, o) partials merged in chunk order by the
// last finishing CTA (deterministic).
#include <cmath>
#include <cstdlib>

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
#ifndef MACE_DTC_STAGES128
#define MACE_DTC_STAGES128 3
#endif
  static constexpr int STAGES = HD >= 128 ? MACE_DTC_STAGES128 : 3;  // hd 64: 2 CTAs per SM; hd 128: 1 (C4: 3 stages 0.49 of HBM, 2 stages 0.33)
  static constexpr int Q_OFF = STAGES * 2 * TILE;       // 2 x [16 rows][HD] K-major
  static constexpr int Q_BYTES = KATOMS * 16 * SWZ;
  static constexpr int P_OFF = Q_OFF + 2 * Q_BYTES;     // 2 x P^T [16 rows][128 tok] K-major SW128
  static constexpr int P_BYTES = 2 * 16 * 128;
  static constexpr int RED_OFF = P_OFF + 2 * P_BYTES;   // float [2][4][16] max, [4][16] sums
  static constexpr int BAR_OFF = RED_OFF + 3 * 4 * 16 * 4;
  static constexpr int N_BARS = 2 * STAGES + 12;
  static constexpr int SMEM = BAR_OFF + N_BARS * 8 + 16 + 1024;
  static constexpr int PARTIAL(int G) { return 2 * G + G * HD; }
};

struct DecItem {  // page-slot range of one item, computed identically by every role
  int seq, h, chunk, nch, pbase, slot, n_pv, npp, kvh, d0, db, de, r0, s0, s1;
};

// SPLIT = 1: the S = K.Q^T MMAs and the O = V^T.P MMAs are issued by two threads in different warps (warp 5 and
// warp 6), so P.V(t) -- and with it the release of tile t's K / V stage -- goes out the moment the softmax publishes
// P(t), instead of queueing behind the arrival of tile t+1 for S(t+1) in a single issuer's program order. Each
// issuer's tcgen05.commit tracks only its own MMAs; the two streams touch disjoint TMEM columns.
template <int HD, int G, int SPLIT>
__global__ void __launch_bounds__(SPLIT ? 224 : 192, 1) attn_decode_tc_kernel(
    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
    const __grid_constant__ CUtensorMap qmap, const MaceSeq* __restrict__ seqs, const int4* __restrict__ items,
    int n_items, const MaceKvLayout kv, int Hq, int Hkv, float scale_log2, __nv_bfloat16* __restrict__ out,
    float* __restrict__ head_norm, float* __restrict__ partials, int* __restrict__ counters) {
  using C = DecTc<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* red_max = reinterpret_cast<float*>(smem + C::RED_OFF);  // [2][4][16]
  float* red_sum = red_max + 2 * 4 * 16;                           // [4][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = bars;                    // [STAGES]
  uint64_t* empty = full + C::STAGES;       // [STAGES]
  uint64_t* qfull = empty + C::STAGES;      // [2]
  uint64_t* qempty = qfull + 2;             // [2]
  uint64_t* sfull = qempty + 2;             // [2]
  uint64_t* sempty = sfull + 2;             // [2]
  uint64_t* pfull = sempty + 2;             // [2]
  uint64_t* ofull = pfull + 2;              // [2]  (pempty == ofull: P(t) is free once P.V(t) completed)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::N_BARS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NT = SPLIT ? 224 : 192;

  // ---- setup: zero V stages, Q and P (skipped page slots / padded heads multiply as finite zeros)
  for (int s = 0; s < C::STAGES; ++s)
    for (int i = tid * 16; i < C::TILE; i += NT * 16)
      *reinterpret_cast<uint4*>(smem + (2 * s + 1) * C::TILE + i) = make_uint4(0, 0, 0, 0);
  for (int i = C::Q_OFF + tid * 16; i < C::RED_OFF; i += NT * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&qfull[b], 1);
      mbar_init(&qempty[b], 1);
      mbar_init(&sfull[b], 1);
      mbar_init(&sempty[b], 4);
      mbar_init(&pfull[b], 4);
      mbar_init(&ofull[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<64>(tmem_slot);
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S[0] 0..15, S[1] 16..31, O[0] 32..47, O[1] 48..63
  pdl_wait();
  pdl_trigger();

  auto item_info = [&](int idx) {
    const int4 it = items[idx];
    const MaceSeq sq = seqs[it.x];
    DecItem d;
    d.seq = it.x;
    d.h = it.y;
    d.chunk = it.z >> 16;
    d.nch = it.z & 0xffff;
    d.pbase = it.w;
    d.slot = sq.slot;
    d.n_pv = sq.n_pv;
    d.npp = (d.n_pv + 15) / 16;
    d.kvh = sq.slot * Hkv + d.h;
    d.d0 = kv.dec_first[d.kvh];
    d.db = kv.dec_base[d.kvh];
    d.de = kv.dec_end[sq.slot];
    d.r0 = (d.d0 - d.db) / 16;
    const int ndp = d.de > d.d0 ? ((d.de - 1 - d.db) / 16 - d.r0 + 1) : 0;
    const int per = (d.npp + d.nch - 1) / d.nch;
    d.s0 = min(d.npp, d.chunk * per);
    d.s1 = d.chunk == d.nch - 1 ? d.npp + ndp : min(d.npp, d.s0 + per);
    return d;
  };
  auto slot_info = [&](const DecItem& d, int p, int& page, int& lo, int& hi) {  // p: page slot in the chunk
    const int ps = d.s0 + p;
    if (ps >= d.s1) {
      page = -1;
      lo = hi = 0;
    } else if (ps < d.npp) {
      page = kv.ptab[(size_t)d.slot * kv.max_prompt_pages + ps] * Hkv + d.h;
      lo = 0;
      hi = min(16, d.n_pv - 16 * ps);
    } else {
      const int r = d.r0 + (ps - d.npp);
      page = kv.dtab[(size_t)d.kvh * kv.max_dec_pages + r];
      const int b = d.db + 16 * r;
      lo = max(0, d.d0 - b);
      hi = min(16, d.de - b);
    }
  };

  if (warp == 4) {
    // ================================================================ producer (TMA)
    // The whole warp: lane q < 8 resolves page slot q of a tile (page-table loads of the 8 slots in parallel,
    // one tile ahead, so their L2 round trip overlaps the ring wait and the previous tile's TMA issue), lane 0
    // arms the stage barrier, every lane with a live page issues its own K / V boxes. (ncu, one lane resolving
    // 8 slots in sequence: 8 dependent L2 round trips per 128-token tile bounded the kernel.)
    uint32_t t = 0, it_local = 0;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++it_local) {
      const DecItem d = item_info(idx);
      const int qb = it_local & 1;
      if (lane == 0) {
        mbar_wait(&qempty[qb], ((it_local >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qfull[qb], C::KATOMS * G * C::SWZ);
        const int qrow = seqs[d.seq].q_start * (Hq + 2 * Hkv) + d.h * G;
#pragma unroll
        for (int a = 0; a < C::KATOMS; ++a)
          tma_load_2d(smem + C::Q_OFF + qb * C::Q_BYTES + a * 16 * C::SWZ, &qmap, &qfull[qb], a * C::ATOM, qrow);
      }
      const int n_tiles = (d.s1 - d.s0 + 7) / 8;
      int pg_next = -1, lo, hi;
      if (lane < 8) slot_info(d, lane, pg_next, lo, hi);
      for (int j = 0; j < n_tiles; ++j, ++t) {
        const int st = t % C::STAGES;
        const int pg = pg_next;
        if (lane < 8 && j + 1 < n_tiles) slot_info(d, 8 * (j + 1) + lane, pg_next, lo, hi);
        const uint32_t live = __ballot_sync(0xffffffffu, lane < 8 && pg >= 0);
        if (lane == 0) {
          mbar_wait(&empty[st], ((t / C::STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], __popc(live) * 2 * C::KATOMS * 16 * C::SWZ);
        }
        __syncwarp();
        if (lane < 8 && pg >= 0) {
          uint8_t* ks = smem + 2 * st * C::TILE;
#pragma unroll
          for (int a = 0; a < C::KATOMS; ++a) {
            tma_load_2d(ks + a * C::ATOM_BYTES + lane * 16 * C::SWZ, &kmap, &full[st], a * C::ATOM, pg * 16);
            tma_load_2d(ks + C::TILE + a * C::ATOM_BYTES + lane * 16 * C::SWZ, &vmap, &full[st], a * C::ATOM,
                        pg * 16);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ================================================================ MMA issuer (single thread)
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 16, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, 16, true, false);
      constexpr uint32_t lbo_v = C::KATOMS > 1 ? C::ATOM_BYTES : 0;  // M=128 pads head dims (re-read atom)
      auto issue_pv = [&](uint32_t tp) {  // P.V of global tile tp
        const int pb = tp & 1;
        mbar_wait(&pfull[pb], (tp >> 1) & 1);
        // O[pb] free: the softmax consumed O(tp-2) before publishing P(tp) (program order), so no wait
        tc_fence_after();
        const uint32_t va = smem_u32(smem + (2 * (tp % C::STAGES) + 1) * C::TILE);
        const uint32_t pa = smem_u32(smem + C::P_OFF + pb * C::P_BYTES);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = smem_desc(va + k * 16 * C::SWZ, lbo_v, 8 * C::SWZ, C::LAYOUT);
          const uint64_t bd = smem_desc(pa + (k / 4) * (16 * 128) + (k % 4) * 32, 16, 1024, 2u);
          umma_bf16(tmem + 32 + pb * 16, ad, bd, idesc_o, k > 0 ? 1u : 0u);
        }
        umma_commit(&ofull[pb]);
        umma_commit(&empty[tp % C::STAGES]);
      };
      uint32_t t = 0, it_local = 0;
      for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++it_local) {
        const DecItem d = item_info(idx);
        const int qb = it_local & 1;
        mbar_wait(&qfull[qb], (it_local >> 1) & 1);
        const int n_tiles = (d.s1 - d.s0 + 7) / 8;
        const uint32_t qa = smem_u32(smem + C::Q_OFF + qb * C::Q_BYTES);
        for (int j = 0; j < n_tiles; ++j, ++t) {
          const int st = t % C::STAGES, sb = t & 1;
          mbar_wait(&full[st], (t / C::STAGES) & 1);
          mbar_wait(&sempty[sb], ((t >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(smem + 2 * st * C::TILE);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const int a = (k * 16) / C::ATOM, off = ((k * 16) % C::ATOM) * 2;
            const uint64_t ad = smem_desc(ka + a * C::ATOM_BYTES + off, 16, 8 * C::SWZ, C::LAYOUT);
            const uint64_t bd = smem_desc(qa + a * 16 * C::SWZ + off, 16, 8 * C::SWZ, C::LAYOUT);
            umma_bf16(tmem + sb * 16, ad, bd, idesc_s, k > 0 ? 1u : 0u);
          }
          umma_commit(&sfull[sb]);
          if (j == n_tiles - 1) umma_commit(&qempty[qb]);
          if (!SPLIT && t > 0) issue_pv(t - 1);
        }
      }
      if (!SPLIT && t > 0) issue_pv(t - 1);
    }
  } else if (warp == 6) {
    // ================================================================ P.V issuer (SPLIT only)
    if (SPLIT && lane == 0) {
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, 16, true, false);
      constexpr uint32_t lbo_v = C::KATOMS > 1 ? C::ATOM_BYTES : 0;
      uint32_t tp = 0;
      for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
        const DecItem d = item_info(idx);
        const int n_tiles = (d.s1 - d.s0 + 7) / 8;
        for (int j = 0; j < n_tiles; ++j, ++tp) {
          const int pb = tp & 1;
          mbar_wait(&pfull[pb], (tp >> 1) & 1);  // P(tp) published => S(tp) done => stage tp's K / V landed
          tc_fence_after();
          const uint32_t va = smem_u32(smem + (2 * (tp % C::STAGES) + 1) * C::TILE);
          const uint32_t pa = smem_u32(smem + C::P_OFF + pb * C::P_BYTES);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t ad = smem_desc(va + k * 16 * C::SWZ, lbo_v, 8 * C::SWZ, C::LAYOUT);
            const uint64_t bd = smem_desc(pa + (k / 4) * (16 * 128) + (k % 4) * 32, 16, 1024, 2u);
            umma_bf16(tmem + 32 + pb * 16, ad, bd, idesc_o, k > 0 ? 1u : 0u);
          }
          umma_commit(&ofull[pb]);
          umma_commit(&empty[tp % C::STAGES]);
        }
      }
    }
  } else {
    // ================================================================ softmax + epilogue (warps 0-3)
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const int q = tid >> 4, row = tid & 15;  // token of the tile: page slot q, row in page
    const int r = tid;                       // head dim owned when folding P.V (< HD)
    uint32_t t = 0;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
      const DecItem d = item_info(idx);
      const int n_tiles = (d.s1 - d.s0 + 7) / 8;
      float m_run[G], l_warp[G], o_acc[G], a_prev[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        m_run[g] = -INFINITY;
        l_warp[g] = 0.f;
        o_acc[g] = 0.f;
        a_prev[g] = 1.f;
      }
      for (int j = 0; j < n_tiles; ++j, ++t) {
        const int sb = t & 1;
        int pg, lo, hi;
        slot_info(d, 8 * j + q, pg, lo, hi);
        const bool valid = pg >= 0 && row >= lo && row < hi;
        mbar_wait(&sfull[sb], (t >> 1) & 1);
        tc_fence_after();
        uint32_t sr[16];
        tmem_ld_32x32b_x16(tmem + sb * 16 + lane_base, sr);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sb]);
        float sv[G];
        float* rm = red_max + (t & 1) * 64;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          sv[g] = valid ? __uint_as_float(sr[g]) * scale_log2 : -INFINITY;
          const float mx = warp_max(sv[g]);
          if (lane == 0) rm[warp * 16 + g] = mx;
        }
        named_bar_sync(1, 128);
        float alpha[G];
        uint8_t* pbuf = smem + C::P_OFF + sb * C::P_BYTES;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float mt = fmaxf(fmaxf(rm[g], rm[16 + g]), fmaxf(rm[32 + g], rm[48 + g]));
          const float mn = fmaxf(m_run[g], mt);
          alpha[g] = (m_run[g] == -INFINITY) ? (mn == -INFINITY ? 1.f : 0.f) : exp2f(m_run[g] - mn);
          m_run[g] = mn;
          const float p = valid ? exp2f(sv[g] - mn) : 0.f;
          l_warp[g] = l_warp[g] * alpha[g] + warp_sum(p);
          const int ch = ((tid & 63) >> 3) ^ (g & 7);
          *reinterpret_cast<__nv_bfloat16*>(pbuf + (tid >> 6) * (16 * 128) + g * 128 + ch * 16 + (tid & 7) * 2) =
              __float2bfloat16(p);
        }
        // P(t) may only be written once P.V(t-2) finished reading this buffer: guaranteed, because the
        // fold of O(t-2) below (previous iteration) waited on ofull of that very MMA
        fence_proxy_async_shared();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[sb]);
        if (j > 0) {  // fold P.V of the previous tile of this item
          const uint32_t tp = t - 1;
          mbar_wait(&ofull[tp & 1], (tp >> 1) & 1);
          tc_fence_after();
          uint32_t orr[16];
          tmem_ld_32x32b_x16(tmem + 32 + (tp & 1) * 16 + lane_base, orr);
          tmem_ld_wait();
#pragma unroll
          for (int g = 0; g < G; ++g) o_acc[g] = o_acc[g] * a_prev[g] + __uint_as_float(orr[g]);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) a_prev[g] = alpha[g];
      }
      {  // fold the item's last tile
        const uint32_t tp = t - 1;
        mbar_wait(&ofull[tp & 1], (tp >> 1) & 1);
        tc_fence_after();
        uint32_t orr[16];
        tmem_ld_32x32b_x16(tmem + 32 + (tp & 1) * 16 + lane_base, orr);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < G; ++g) o_acc[g] = o_acc[g] * a_prev[g] + __uint_as_float(orr[g]);
      }
      // ---- l across warps
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (lane == 0) red_sum[warp * 16 + g] = l_warp[g];
      named_bar_sync(1, 128);
      float l_tot[G];
#pragma unroll
      for (int g = 0; g < G; ++g) l_tot[g] = (red_sum[g] + red_sum[16 + g]) + (red_sum[32 + g] + red_sum[48 + g]);
      const int orow = seqs[d.seq].q_start;
      auto emit = [&](const float* l_, const float* o_) {
        float nv[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float inv = l_[g] > 0.f ? 1.f / l_[g] : 0.f;
          const float v = o_[g] * inv;
          if (r < HD) out[(size_t)orow * Hq * HD + (size_t)(d.h * G + g) * HD + r] = __float2bfloat16(v);
          nv[g] = warp_sum(r < HD ? v * v : 0.f);
        }
        if (head_norm) {
          named_bar_sync(1, 128);  // red_sum reads above are done before reuse
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (lane == 0) red_sum[warp * 16 + g] = nv[g];
          named_bar_sync(1, 128);
          if (tid < G)
            head_norm[(size_t)orow * Hq + d.h * G + tid] =
                sqrtf((red_sum[tid] + red_sum[16 + tid]) + (red_sum[32 + tid] + red_sum[48 + tid]));
        }
      };
      if (d.nch == 1) {
        emit(l_tot, o_acc);
      } else {
        float* mine = partials + (size_t)(d.pbase + d.chunk) * C::PARTIAL(G);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (tid == 0) {
            mine[g] = m_run[g];
            mine[G + g] = l_tot[g];
          }
          if (r < HD) mine[2 * G + g * HD + r] = o_acc[g];
        }
        __threadfence();
        named_bar_sync(1, 128);
        int* flag = reinterpret_cast<int*>(red_sum + 63);
        if (tid == 0) *flag = atomicAdd(&counters[d.kvh], 1);
        named_bar_sync(1, 128);
        const bool last = *flag == d.nch - 1;
        if (last) {
          __threadfence();
          const float* first = partials + (size_t)d.pbase * C::PARTIAL(G);
          float L[G], A[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            float M = -INFINITY;
            for (int c = 0; c < d.nch; ++c) M = fmaxf(M, __ldcg(first + c * C::PARTIAL(G) + g));
            L[g] = 0.f;
            A[g] = 0.f;
            for (int c = 0; c < d.nch; ++c) {  // chunk order: deterministic
              const float* pc = first + c * C::PARTIAL(G);
              const float mc = __ldcg(pc + g);
              const float sc = mc == -INFINITY ? 0.f : exp2f(mc - M);
              L[g] += __ldcg(pc + G + g) * sc;
              if (r < HD) A[g] += __ldcg(pc + 2 * G + g * HD + r) * sc;
            }
          }
          emit(L, A);
          if (tid == 0) counters[d.kvh] = 0;
        }
      }
      named_bar_sync(1, 128);  // red buffers reusable by the next item
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<64>(tmem);
  }
}

static bool encode_rows(MaceCtx* ctx, CUtensorMap* m, const void* base, long long rows, int HD, int box_rows, int atom,
                        int swz) {
  cuuint64_t dims[2] = {(cuuint64_t)HD, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)HD * 2};
  cuuint32_t box[2] = {(cuuint32_t)atom, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return ctx->encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD, int G, int SPLIT>
int launch_decode_tc(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s) {
  using C = DecTc<HD>;
  CUtensorMap km, vm, qm;
  // qkv viewed as [T * (Hq + 2Hkv) head rows, HD]: the G query rows of a group are one box
  if (!encode_rows(ctx, &km, a->k_pool, a->pool_pages * 16, HD, 16, C::ATOM, C::SWZ) ||
      !encode_rows(ctx, &vm, a->v_pool, a->pool_pages * 16, HD, 16, C::ATOM, C::SWZ) ||
      !encode_rows(ctx, &qm, a->qkv, (long long)a->T * (a->Hq + 2 * a->Hkv), HD, G, C::ATOM, C::SWZ))
    return mace_fail(ctx, MACE_ERR_LAUNCH, "attn decode tc: tensor map encode failed");
  const size_t need = (size_t)a->n_dec * C::PARTIAL(G) * 4;
  if (!a->dec_workspace || a->dec_workspace_bytes < need || !a->dec_counters)
    return mace_fail(ctx, MACE_ERR_ARG, "attn decode: workspace/counters too small");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_tc_kernel<HD, G, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  const int per_sm = (227 * 1024) / C::SMEM;
  int grid = ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  if (grid > a->n_dec) grid = a->n_dec;
  launch_k(attn_decode_tc_kernel<HD, G, SPLIT>, grid, SPLIT ? 224 : 192, C::SMEM, s, km, vm, qm, a->seqs,
           reinterpret_cast<const int4*>(a->dec_items), a->n_dec, a->kv, a->Hq, a->Hkv, sl2, (__nv_bfloat16*)a->out,
           a->head_norm, (float*)a->dec_workspace, a->dec_counters);
  ctx->launches++;
  return 0;
}

int dispatch_decode_tc(MaceCtx* ctx, const MaceAttnArgs* a, float sl2, cudaStream_t s) {
  const int G = a->Hq / a->Hkv;
  // MACE_DTC_ISSUE=1: one MMA issuer (S and P.V in one thread's program order); default 2 (split issuers)
  static const int split = [] {
    const char* e = getenv("MACE_DTC_ISSUE");
    return (e && atoi(e) == 1) ? 0 : 1;
  }();
#define MACE_DTC_G(HD_, G_) \
  return split ? launch_decode_tc<HD_, G_, 1>(ctx, a, sl2, s) : launch_decode_tc<HD_, G_, 0>(ctx, a, sl2, s);
#define MACE_DTC(HD_)                                                 \
  switch (G) {                                                        \
    case 1: MACE_DTC_G(HD_, 1)                                        \
    case 2: MACE_DTC_G(HD_, 2)                                        \
    case 4: MACE_DTC_G(HD_, 4)                                        \
    case 8: MACE_DTC_G(HD_, 8)                                        \
    default: return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn decode: GQA group must be 1, 2, 4 or 8"); \
  }
  switch (a->hd) {
    case 32: MACE_DTC(32)
    case 64: MACE_DTC(64)
    case 128: MACE_DTC(128)
    default: return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "attn decode: head_dim must be 32, 64 or 128");
  }
#undef MACE_DTC
#undef MACE_DTC_G
}

}  // namespace mace
