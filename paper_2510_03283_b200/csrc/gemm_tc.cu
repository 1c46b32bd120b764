// bf16 tcgen05 GEMM for sm_100a: C[M,N] = alpha * A[M,K] . B[N,K]^T  (+bias, +=C, split-K)
//
// Replaces the cost-model stand-in for the packed QKV / O / MLP / lm_head projections of the
// hybrid iteration (reference: engine.py:588-600 charges prefill/decode/FT latency from
// cost_model.get_workload, cost_model.py:92-106) and their backward on fine-tune rows.
//
// Design (B200-first):
//  * persistent, one CTA per SM, static tile schedule (tile = blockIdx.x + i * gridDim.x)
//  * warp 0: TMA producer (cp.async.bulk.tensor, 128B swizzle) over a kStages smem ring
//  * warp 1: single-thread tcgen05.mma issuer (M=128, N=BN, K=16 per instruction)
//  * warp 2: TMEM allocator (2 accumulator buffers -> epilogue of tile i overlaps MMA of i+1)
//  * warps 4..7: epilogue, tcgen05.ld 32x32b -> registers -> fused bias / residual / convert
//  * operands may be K-major (row-major [rows, K]) or MN-major (row-major [K, rows]); the MN-major
//    form is what the fine-tune backward needs (dX = dY.W and dW = dY^T.X) without transposes.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "mace_internal.h"

namespace mace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K

template <int BN>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;  // 16 KB
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // epilogue staging for the TMA-store path: 4 warps x 2 buffers x (32 rows x 128 B)
  static constexpr int kCBytes = 4 * 2 * 4096;
  static constexpr int kBudget = 227 * 1024 - kCBytes - 1024 /*align*/ - 256 /*barriers*/;
  static constexpr int kStages = kBudget / kStageBytes > 8 ? 8 : kBudget / kStageBytes;
  static constexpr int kTmemCols = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kStages * kStageBytes + kCBytes + 1024 + 256;
};

struct GemmParams {
  int M, N, K;
  int num_m, num_n, splits, kb_total, kb_per_split;
  int c_reduce;  // TMA epilogue: 1 -> global += tile (cp.reduce.async.bulk .add)
  int c_slab;    // TMA epilogue: 1 -> per-split fp32 slabs through a 3-D map {N, M, splits}
  int dbg;       // trace builds only (tools/gemm_trace.py probes); 0 otherwise
  int b_static;  // B not written by the preceding kernel: first ring of B tiles loads before the PDL wait
  int stages;    // smem ring depth of the single-CTA kernel
  int swiglu;    // EPI_BF16_SWIGLU: a BN tile = BN/2 gate rows (row n) + BN/2 up rows (row N + n) of B
  GemmEpilogue ep;
};


// Epilogue chunk of one warp (32 rows) through smem and a TMA store: registers -> 128B-swizzled
// [32 rows][128 B] staging (conflict-free: 16-byte chunk q of row r lives at q ^ (r & 7)) ->
// cp.async.bulk.tensor store (or .add reduction) of a {cols, 32 rows} box. Coalesced, asynchronous,
// bounds-clipped by the tensor map, so the epilogue no longer issues 32 row-strided stores per warp.
MACE_DEV void stage_row_chunk16(uint8_t* st, uint32_t lane, int q, uint4 w) {
  *reinterpret_cast<uint4*>(st + lane * 128 + ((q ^ (lane & 7)) << 4)) = w;
}

// silu(gate) * up for the fused Llama MLP epilogue (fp32 accumulators, one bf16 rounding of the product)
// silu(g) * u with a branch-free reciprocal: the IEEE division's special-case branch kept the epilogue warps (one
// per SM sub-partition) from overlapping the 64 independent evaluations of a chunk -- the SwiGLU epilogue took
// 18.7 us of a 33.8 us decode-sized (M = 256) up projection (tools/gemm_trace.py; plain bf16 epilogue: 1.8 us)
MACE_DEV float swiglu_f(float g, float u) { return g * __fdividef(1.f, 1.f + __expf(-g)) * u; }

// fused SwiGLU epilogue of one tile (both GEMM kernels): this warp's 32 rows, TMEM columns [0, BN/2) hold
// the gate projection and [BN/2, BN) the up projection of the same BN/2 outputs; two 64-column chunks are
// staged in the warp's two 4 KB buffers and TMA-stored; the accumulator is released after the last loads
template <int BN>
MACE_DEV void swiglu_epilogue(const CUtensorMap* map_c, uint8_t* smem_c, uint32_t t_row, int quarter, int lane,
                              int row0, int col_base, int N, uint64_t* tempty, bool remote, uint32_t tempty_cluster) {
  constexpr int HALF = BN / 2;
#pragma unroll 1
  for (int oc = 0; oc < HALF; oc += 64) {
    uint32_t r[128];
    tmem_ld_32x32b_x32(t_row + oc, *reinterpret_cast<uint32_t(*)[32]>(r));
    tmem_ld_32x32b_x32(t_row + oc + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
    tmem_ld_32x32b_x32(t_row + HALF + oc, *reinterpret_cast<uint32_t(*)[32]>(r + 64));
    tmem_ld_32x32b_x32(t_row + HALF + oc + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 96));
    tmem_ld_wait();
    if (oc + 64 >= HALF) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (remote) mbar_arrive_cluster(tempty_cluster);
        else mbar_arrive(tempty);
      }
    }
    const int col0 = col_base + oc;
    if (col0 >= N) continue;
    if (lane == 0) bulk_wait_read<1>();
    __syncwarp();
    uint8_t* st = smem_c + (quarter * 2 + ((oc / 64) & 1)) * 4096;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = swiglu_f(__uint_as_float(r[q * 8 + j]), __uint_as_float(r[64 + q * 8 + j]));
      stage_row_chunk16(st, lane, q, make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                                                pack_bf16(v[6], v[7])));
    }
    fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(map_c, st, col0, row0);
      bulk_commit();
    }
  }
}

// fused greedy decode head (EPI_ARGMAX): this thread's accumulator row over the tile's columns -> (largest value,
// first column holding it), in ascending column order; tcgen05.ld is warp-collective, the loop bound is warp-uniform
template <int BN>
MACE_DEV void argmax_row(uint32_t t_row, int col_base, int N, float alpha, float& best, int& bi) {
  best = -INFINITY;
  bi = 0x7fffffff;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    if (col_base + c0 >= N) break;
    uint32_t r[32];
    tmem_ld_32x32b_x32(t_row + c0, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float v = __uint_as_float(r[j]) * alpha;
      if (col_base + c0 + j < N && v > best) {
        best = v;
        bi = col_base + c0 + j;
      }
    }
  }
}

// the row's key: orderable fp32 bits in the high word, the complemented column in the low word, so atomicMax picks
// the largest value and, among equal values, the lowest column (order-independent: deterministic)
MACE_DEV void argmax_publish(unsigned long long* keys, int row, int M, float best, int bi) {
  if (row >= M || bi == 0x7fffffff) return;
  uint32_t b = __float_as_uint(best);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  atomicMax(keys + row, ((unsigned long long)b << 32) | (unsigned long long)(0xffffffffu - (uint32_t)bi));
}

#ifdef MACE_GEMM_TRACE
// phase timestamps (%globaltimer ns) per CTA, tools/gemm_trace.py: [cta][32]
__device__ unsigned long long* g_gemm_trace = nullptr;
__device__ __forceinline__ void trace_at(int slot) {
  if (g_gemm_trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_trace[blockIdx.x * 64 + slot] = t;
    g_gemm_trace[blockIdx.x * 64 + 32 + slot] = clock64();  // SM cycles (same-CTA differences)
  }
}
#define TRACE(slot) trace_at(slot)
static int g_gemm_dbg_host = 0;  // 1: TMA only for the first ring pass (MMA-rate probe), 2: no MMA (TMA-rate probe)
#else
#define TRACE(slot)
#endif

template <int BN, bool A_MN, bool B_MN, bool TMA_EPI>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c, const GemmParams p) {
  using Cfg = GemmCfg<BN>;
  const int S = p.stages;  // ring depth (<= Cfg::kStages; small-K GEMMs use fewer to leave smem for the next kernel)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * Cfg::kABytes;
  uint8_t* smem_c = smem + S * Cfg::kStageBytes;  // epilogue staging (TMA_EPI)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_c + Cfg::kCBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int num_tiles = p.num_m * p.num_n * p.splits;
  if (threadIdx.x == 0) TRACE(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    if (TMA_EPI) tma_prefetch_desc(&map_c);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) TRACE(1);

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (whole warp walks the schedule so
    // every index is warp-uniform and lives in uniform registers; one elected lane issues)
    auto load_b = [&](int stage, int kb, int n_blk) {
      uint8_t* sb = smem_b + stage * Cfg::kBBytes;
      if (!B_MN && p.swiglu) {  // gate rows n*BN/2.. and up rows N + n*BN/2.. of the stacked [2N, K] weight
        tma_load_2d(sb, &map_b, &full_bar[stage], kb * kBK, n_blk * (BN / 2));
        tma_load_2d(sb + (BN / 2) * kBK * 2, &map_b, &full_bar[stage], kb * kBK, p.N + n_blk * (BN / 2));
      } else if (!B_MN) {
        tma_load_2d(sb, &map_b, &full_bar[stage], kb * kBK, n_blk * BN);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 64; ++j)
          tma_load_2d(sb + j * (64 * kBK * 2), &map_b, &full_bar[stage], n_blk * BN + j * 64, kb * kBK);
      }
    };
    // weights (B) do not depend on the preceding kernel: fill the first ring of B tiles while it drains
    int pre = 0;
    if (p.b_static && (int)blockIdx.x < num_tiles) {
      const int t = blockIdx.x;
      const int n_blk = (t / p.num_m) % p.num_n;
      const int kb0 = (t / (p.num_m * p.num_n)) * p.kb_per_split;
      pre = min(S, min(p.kb_total, kb0 + p.kb_per_split) - kb0);
      if (elect_one()) {
        for (int i = 0; i < pre; ++i) {
          mbar_arrive_expect_tx(&full_bar[i], Cfg::kStageBytes);
          load_b(i, kb0 + i, n_blk);
        }
      }
      __syncwarp();
    }
    pdl_wait();
    pdl_trigger();
    if (lane == 0) TRACE(2);
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int m_blk = t % p.num_m;
      const int n_blk = (t / p.num_m) % p.num_n;
      const int split = t / (p.num_m * p.num_n);
      const int kb0 = split * p.kb_per_split;
      const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
#ifdef MACE_GEMM_TRACE
        if (p.dbg == 4 && (kb - kb0) >= S) break;
#endif
        const bool b_done = t == (int)blockIdx.x && kb - kb0 < pre;  // B already in flight (pre-wait)
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (elect_one()) {
#ifdef MACE_GEMM_TRACE
          if ((p.dbg == 1 || p.dbg == 3) && (kb - kb0) >= S) {
            mbar_arrive(&full_bar[stage]);
          } else {
#endif
          if (!b_done) mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          uint8_t* sa = smem_a + stage * Cfg::kABytes;
          if (!A_MN) {
            tma_load_2d(sa, &map_a, &full_bar[stage], kb * kBK, m_blk * kBM);
          } else {
#pragma unroll
            for (int j = 0; j < kBM / 64; ++j)
              tma_load_2d(sa + j * (64 * kBK * 2), &map_a, &full_bar[stage], m_blk * kBM + j * 64, kb * kBK);
          }
#ifdef MACE_GEMM_TRACE
          if (t == (int)blockIdx.x && kb == kb0) TRACE(3);
#endif
          if (!b_done) load_b(stage, kb, n_blk);
#ifdef MACE_GEMM_TRACE
          }
#endif
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (whole warp; one elected lane issues)
    constexpr uint32_t idesc = idesc_bf16_f32(kBM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t a_base = smem_u32(smem_a), b_base = smem_u32(smem_b);
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int split = t / (p.num_m * p.num_n);
      const int kb0 = split * p.kb_per_split;
      const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
#ifdef MACE_GEMM_TRACE
        if (!(p.dbg == 4 && (kb - kb0) >= S))
#endif
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
#ifdef MACE_GEMM_TRACE
        if (lane == 0 && t == (int)blockIdx.x && kb == kb0) TRACE(4);
#endif
        const uint32_t a_addr = a_base + stage * Cfg::kABytes;
        const uint32_t b_addr = b_base + stage * Cfg::kBBytes;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // K-major: advance 16 elems = 32 B inside the swizzle atom; SBO = 8 rows * 128 B.
            // MN-major: advance 16 K-rows = 2048 B; LBO = one 64-wide MN block (64 rows * 128 B).
            const uint64_t ad = A_MN ? smem_desc_sw128(a_addr + k * 2048, 64 * kBK * 2, 1024)
                                     : smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc_sw128(b_addr + k * 2048, 64 * kBK * 2, 1024)
                                     : smem_desc_sw128(b_addr + k * 32, 16, 1024);
#ifdef MACE_GEMM_TRACE
            if (p.dbg == 2) continue;
            if (p.dbg == 3) {  // independent accumulators for odd k (dependency-latency probe)
              umma_bf16(d_tmem + ((k & 1) ? ((acc ^ 1) - acc) * BN : 0), ad, bd, idesc, (kb > kb0 || k > 1) ? 1u : 0u);
              continue;
            }
#endif
            umma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
#ifdef MACE_GEMM_TRACE
          if (!(p.dbg == 4))
#endif
          umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
#ifdef MACE_GEMM_TRACE
      { const int ti = (t - (int)blockIdx.x) / (int)gridDim.x; if (lane == 0 && ti < 5) TRACE(8 + ti * 4); }
#endif
      if (elect_one()) umma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue (128 threads <-> 128 TMEM lanes)
    pdl_wait();  // outputs may be read / accumulated by the preceding kernel
    const uint32_t quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int stage_buf = 0;
    const GemmEpilogue& ep = p.ep;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int m_blk = t % p.num_m;
      const int n_blk = (t / p.num_m) % p.num_n;
      const int split = t / (p.num_m * p.num_n);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
#ifdef MACE_GEMM_TRACE
      const int ti_ = (t - (int)blockIdx.x) / (int)gridDim.x;
      if (warp == 4 && lane == 0 && ti_ < 5) TRACE(8 + ti_ * 4 + 1);
#endif
      if (ep.mode == EPI_ARGMAX) {
        float best;
        int bi;
        argmax_row<BN>(tmem_base + ((quarter * 32u) << 16) + acc * BN, n_blk * BN, p.N, ep.alpha, best, bi);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        argmax_publish(reinterpret_cast<unsigned long long*>(ep.out), m_blk * kBM + quarter * 32 + lane, p.M, best, bi);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      if constexpr (TMA_EPI) {
        if (p.swiglu) {
          swiglu_epilogue<BN>(&map_c, smem_c, tmem_base + ((quarter * 32u) << 16) + acc * BN, quarter, lane,
                              m_blk * kBM + quarter * 32, n_blk * (BN / 2), p.N, &tempty_bar[acc], false, 0);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
          continue;
        }
        // per group of two staged chunks (bf16: 2 x 64 columns, fp32: 2 x 32): every TMEM load of the group is
        // issued before one wait, the accumulator is handed back to the MMA warp as soon as the tile's last
        // group is in registers, and one proxy fence + one commit cover both staging buffers
        const bool bf16_out = ep.mode == EPI_BF16 || ep.mode == EPI_BF16_GELU;
        const bool gelu = ep.mode == EPI_BF16_GELU;
        const int cw = bf16_out ? 64 : 32;  // columns per 128-byte staged row
        const int row0 = m_blk * kBM + quarter * 32;
        const bool add_bias = ep.bias != nullptr && split == 0;
        const uint32_t t_row = tmem_base + ((quarter * 32u) << 16) + acc * BN;
#pragma unroll 1
        for (int g0 = 0; g0 < BN; g0 += 2 * cw) {
          uint32_t r[128];
          tmem_ld_32x32b_x32(t_row + g0, *reinterpret_cast<uint32_t(*)[32]>(r));
          tmem_ld_32x32b_x32(t_row + g0 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
          if (bf16_out && g0 + 64 < BN) {  // BN 64: one bf16 chunk per tile
            tmem_ld_32x32b_x32(t_row + g0 + 64, *reinterpret_cast<uint32_t(*)[32]>(r + 64));
            tmem_ld_32x32b_x32(t_row + g0 + 96, *reinterpret_cast<uint32_t(*)[32]>(r + 96));
          }
          tmem_ld_wait();
          if (g0 + 2 * cw >= BN) {  // the whole tile is in registers: release the accumulator
            tc_fence_before();
            __syncwarp();
#ifdef MACE_GEMM_TRACE
            if (warp == 4 && lane == 0 && ti_ < 5) TRACE(8 + ti_ * 4 + 2);
#endif
            if (lane == 0) mbar_arrive(&tempty_bar[acc]);
          }
          if (lane == 0) bulk_wait_read<0>();  // both staging buffers have been read by the previous group's stores
          __syncwarp();
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int col0 = n_blk * BN + g0 + b * cw;
            if (g0 + b * cw >= BN || col0 >= p.N) break;
            uint8_t* st = smem_c + (quarter * 2 + b) * 4096;
            if (bf16_out) {
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const int c = q * 8 + j;
                  v[j] = __uint_as_float(r[b * 64 + c]) * ep.alpha;
                  if (add_bias && col0 + c < p.N) v[j] += __bfloat162float(ep.bias[col0 + c]);
                  if (gelu) v[j] = gelu_tanh_fast(v[j]);
                }
                stage_row_chunk16(st, lane, q, make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                                                          pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7])));
              }
            } else {
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int c = q * 4 + j;
                  v[j] = __uint_as_float(r[b * 32 + c]) * ep.alpha;
                  if (add_bias && col0 + c < p.N) v[j] += __bfloat162float(ep.bias[col0 + c]);
                }
                stage_row_chunk16(st, lane, q, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                                                          __float_as_uint(v[2]), __float_as_uint(v[3])));
              }
            }
          }
          fence_proxy_async_shared();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int col0 = n_blk * BN + g0 + b * cw;
              if (g0 + b * cw >= BN || col0 >= p.N) break;
              uint8_t* st = smem_c + (quarter * 2 + b) * 4096;
              if (p.c_slab)
                tma_store_3d(&map_c, st, col0, row0, split);
              else if (p.c_reduce)
                tma_reduce_add_2d(&map_c, st, col0, row0);
              else
                tma_store_2d(&map_c, st, col0, row0);
            }
            bulk_commit();
          }
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      const int row = m_blk * kBM + quarter * 32 + lane;
      const bool row_ok = row < p.M;
      const bool add_bias = ep.bias != nullptr && split == 0;
      // deterministic split-K: split s writes its own fp32 slab, reduced later in fixed order
      void* const ep_out = ep.split_stride ? (void*)(reinterpret_cast<float*>(ep.out) + (size_t)split * ep.split_stride)
                                           : ep.out;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((quarter * 32u) << 16) + acc * BN + c0, r);
        tmem_ld_wait();
        const int col0 = n_blk * BN + c0;
        if (!row_ok || col0 >= p.N) continue;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * ep.alpha;
        if (add_bias) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < p.N) v[j] += __bfloat162float(ep.bias[col0 + j]);
        }
        const bool full = (col0 + 32 <= p.N) && ((ep.ldo & 7) == 0);
        if (ep.mode == EPI_BF16_GELU) {  // fused GPT-2 MLP activation (gelu_tanh) on the up projection
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = gelu_tanh_fast(v[j]);
        }
        if (ep.mode == EPI_BF16 || ep.mode == EPI_BF16_GELU) {
          __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(ep_out) + (size_t)row * ep.ldo + col0;
          if (full) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint4 w = make_uint4(pack_bf16(v[j], v[j + 1]), pack_bf16(v[j + 2], v[j + 3]),
                                   pack_bf16(v[j + 4], v[j + 5]), pack_bf16(v[j + 6], v[j + 7]));
              *reinterpret_cast<uint4*>(out + j) = w;
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) out[j] = __float2bfloat16(v[j]);
          }
        } else if (ep.mode == EPI_F32) {
          float* out = reinterpret_cast<float*>(ep_out) + (size_t)row * ep.ldo + col0;
          if (full) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(out + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) out[j] = v[j];
          }
        } else if (ep.mode == EPI_F32_ADD) {
          // out += v (exclusive owner of the tile: plain read-modify-write)
          float* out = reinterpret_cast<float*>(ep.out) + (size_t)row * ep.ldo + col0;
          if (full) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 o = *reinterpret_cast<float4*>(out + j);
              o.x += v[j]; o.y += v[j + 1]; o.z += v[j + 2]; o.w += v[j + 3];
              *reinterpret_cast<float4*>(out + j) = o;
            }
          } else {
            for (int j = 0; j < 32 && col0 + j < p.N; ++j) out[j] += v[j];
          }
        } else {  // EPI_F32_ATOMIC: split-K partials / shared accumulation
          float* out = reinterpret_cast<float*>(ep.out) + (size_t)row * ep.ldo + col0;
          for (int j = 0; j < 32 && col0 + j < p.N; ++j) atomicAdd(out + j, v[j]);
        }
      }
      tc_fence_before();
      __syncwarp();
#ifdef MACE_GEMM_TRACE
      if (warp == 4 && lane == 0 && ti_ < 5) TRACE(8 + ti_ * 4 + 2);
#endif
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  // the staging smem must outlive the stores' reads; their global writes complete with the grid (the dependent
  // kernel's griddepcontrol.wait orders after them), so the CTA does not wait for the write round trip
  if (TMA_EPI && warp >= 4 && lane == 0) bulk_wait_read<0>();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
  if (threadIdx.x == 0) TRACE(31);
}

// ====================================================================================================
// CTA-pair GEMM (cta_group::2) for the large prefill / fine-tune projections.
//
// A single-CTA 128 x 256 tile is shared-memory-bound on B200: per K=16 step the MMA reads 12 KB of operands
// from smem while TMA writes the next 12 KB, ~192 B/clk against ~128 B/clk of smem bandwidth, which caps it
// near 65% of the tensor peak. A CTA pair (two SMs of one TPC, cluster of 2) computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 issued by the leader: each CTA stages only its 128 rows of A and its BN/2 rows of
// B, so per-SM operand traffic halves at the same MMA rate. Roles (256 threads per CTA):
//   warp 0 (both CTAs): TMA producer; both CTAs' loads complete on the LEADER's full barrier
//   warp 1 (leader):    single-thread MMA issue; commits multicast to both CTAs' empty / tmem-full barriers
//   warp 2 (both):      TMEM allocation (cta_group::2: one warp of each CTA)
//   warps 4..7 (both):  epilogue of the CTA's 128 accumulator rows (TMA-store), then a cluster-scope arrive
//                       on the leader's tmem-empty barrier (8 arrivals = 4 warps x 2 CTAs)
// Tiles are walked in groups of kGroupM m-tiles (n outer within a group) so the ~74 tiles in flight share
// A and B panels through L2.
// ====================================================================================================
template <int BN>
struct Gemm2Cfg {
  static constexpr int kABytes = 128 * kBK * 2;           // this CTA's 128 rows of A
  static constexpr int kBBytes = (BN / 2) * kBK * 2;      // this CTA's BN/2 rows of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kCBytes = 4 * 2 * 4096;
  static constexpr int kBudget = 227 * 1024 - kCBytes - 1024 - 256;
#ifndef MACE_GEMM2_MAX_STAGES
#define MACE_GEMM2_MAX_STAGES 8
#endif
  static constexpr int kStages = kBudget / kStageBytes > MACE_GEMM2_MAX_STAGES ? MACE_GEMM2_MAX_STAGES : kBudget / kStageBytes;
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kStages * kStageBytes + kCBytes + 1024 + 256;
};
#ifndef MACE_GEMM_GROUP_M
#define MACE_GEMM_GROUP_M 16  // sweep override (-D)
#endif
constexpr int kGroupM = MACE_GEMM_GROUP_M;

MACE_DEV void tile2_coords(int t, int num_m, int num_n, int& m_blk, int& n_blk) {
  const int group = t / (kGroupM * num_n);
  const int first_m = group * kGroupM;
  const int gm = min(kGroupM, num_m - first_m);
  const int r = t - group * kGroupM * num_n;
  m_blk = first_m + r % gm;
  n_blk = r / gm;
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_c, const GemmParams p) {
  using Cfg = Gemm2Cfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * Cfg::kABytes;
  uint8_t* smem_c = smem + S * Cfg::kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_c + Cfg::kCBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int num_tiles = p.num_m * p.num_n;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    tma_prefetch_desc(&map_c);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any cross-CTA arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    auto load_b = [&](int stage, int kb, int n_blk, uint32_t bar) {
      // swiglu: the leader holds the gate rows, the peer the up rows of the same BN/2 outputs
      const int row = p.swiglu ? (rank ? p.N : 0) + n_blk * (BN / 2) : n_blk * BN + rank * (BN / 2);
      if constexpr (B_MN) {  // [K, N] storage: this CTA's BN/2 columns as 64-wide MN blocks
#pragma unroll
        for (int j = 0; j < BN / 128; ++j)
          tma_load_2d_pair(smem_b + stage * Cfg::kBBytes + j * (64 * kBK * 2), &map_b, bar, row + j * 64, kb * kBK);
      } else {
        tma_load_2d_pair(smem_b + stage * Cfg::kBBytes, &map_b, bar, kb * kBK, row);
      }
    };
    auto load_a = [&](int stage, int kb, int m_blk, uint32_t bar) {
      const int row = m_blk * 256 + rank * 128;
      if constexpr (A_MN) {  // [K, M] storage: this CTA's 128 rows as two 64-wide MN blocks
#pragma unroll
        for (int j = 0; j < 2; ++j)
          tma_load_2d_pair(smem_a + stage * Cfg::kABytes + j * (64 * kBK * 2), &map_a, bar, row + j * 64, kb * kBK);
      } else {
        tma_load_2d_pair(smem_a + stage * Cfg::kABytes, &map_a, bar, kb * kBK, row);
      }
    };
    const uint32_t full0 = mapa_shared(smem_u32(&full_bar[0]), 0);  // leader's full barriers
    int pre = 0;
    if (p.b_static && cid < num_tiles) {
      int m_blk, n_blk;
      tile2_coords(cid, p.num_m, p.num_n, m_blk, n_blk);
      pre = min(S, p.kb_total);
      if (elect_one()) {
        for (int i = 0; i < pre; ++i) {
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[i], 2 * Cfg::kStageBytes);
          load_b(i, i, n_blk, full0 + i * 8);
        }
      }
      __syncwarp();
    }
    pdl_wait();
    pdl_trigger();
    int stage = 0;
    uint32_t phase = 0;
    for (int t = cid; t < num_tiles; t += ncl) {
      int m_blk, n_blk;
      tile2_coords(t, p.num_m, p.num_n, m_blk, n_blk);
      for (int kb = 0; kb < p.kb_total; ++kb) {
        const bool b_done = t == cid && kb < pre;
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (elect_one()) {
          const uint32_t bar = full0 + stage * 8;
          if (rank == 0 && !b_done) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::kStageBytes);
          load_a(stage, kb, m_blk, bar);
          if (!b_done) load_b(stage, kb, n_blk, bar);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ------------------------------------------------ MMA issuer (leader only)
    constexpr uint32_t idesc = idesc_bf16_f32(256, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t a_base = smem_u32(smem_a), b_base = smem_u32(smem_b);
    for (int t = cid; t < num_tiles; t += ncl) {
      mbar_wait_cluster(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < p.kb_total; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint32_t a_addr = a_base + stage * Cfg::kABytes;
        const uint32_t b_addr = b_base + stage * Cfg::kBBytes;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // K-major: 16 K-elements = 32 B inside the swizzle atom; MN-major: 16 K-rows = 2048 B, LBO = one
            // 64-wide MN block (as in the single-CTA kernel)
            const uint64_t ad = A_MN ? smem_desc_sw128(a_addr + k * 2048, 64 * kBK * 2, 1024)
                                     : smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc_sw128(b_addr + k * 2048, 64 * kBK * 2, 1024)
                                     : smem_desc_sw128(b_addr + k * 32, 16, 1024);
            umma_bf16_pair(d_tmem, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit_pair(&empty_bar[stage], 0x3);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) umma_commit_pair(&tfull_bar[acc], 0x3);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue (both CTAs: this CTA's 128 rows)
    pdl_wait();
    const uint32_t quarter = warp & 3;
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int stage_buf = 0;
    const GemmEpilogue& ep = p.ep;
    const bool bf16_out = ep.mode == EPI_BF16 || ep.mode == EPI_BF16_GELU;
    const int cw = bf16_out ? 64 : 32;
    for (int t = cid; t < num_tiles; t += ncl) {
      int m_blk, n_blk;
      tile2_coords(t, p.num_m, p.num_n, m_blk, n_blk);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row0 = m_blk * 256 + rank * 128 + quarter * 32;
      if (ep.mode == EPI_ARGMAX) {
        float best;
        int bi;
        argmax_row<BN>(tmem_base + ((quarter * 32u) << 16) + acc * BN, n_blk * BN, p.N, ep.alpha, best, bi);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
        argmax_publish(reinterpret_cast<unsigned long long*>(ep.out), row0 + lane, p.M, best, bi);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      if (p.swiglu) {
        swiglu_epilogue<BN>(&map_c, smem_c, tmem_base + ((quarter * 32u) << 16) + acc * BN, quarter, lane, row0,
                            n_blk * (BN / 2), p.N, nullptr, true, tempty0 + acc * 8);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += cw) {
        const int col0 = n_blk * BN + c0;
        if (col0 >= p.N) break;
        uint32_t r[64];
        const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + acc * BN + c0;
        tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
        if (bf16_out) tmem_ld_32x32b_x32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        tmem_ld_wait();
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        uint8_t* st = smem_c + (quarter * 2 + stage_buf) * 4096;
        if (bf16_out) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int c = q * 8 + j;
              v[j] = __uint_as_float(r[c]) * ep.alpha;
              if (ep.bias != nullptr && col0 + c < p.N) v[j] += __bfloat162float(ep.bias[col0 + c]);
              if (ep.mode == EPI_BF16_GELU) v[j] = gelu_tanh_fast(v[j]);
            }
            stage_row_chunk16(st, lane, q, make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                                                      pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7])));
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int c = q * 4 + j;
              v[j] = __uint_as_float(r[c]) * ep.alpha;
              if (ep.bias != nullptr && col0 + c < p.N) v[j] += __bfloat162float(ep.bias[col0 + c]);
            }
            stage_row_chunk16(st, lane, q, make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                                                      __float_as_uint(v[2]), __float_as_uint(v[3])));
          }
        }
        fence_proxy_async_shared();
        __syncwarp();
        if (lane == 0) {
          if (p.c_reduce)
            tma_reduce_add_2d(&map_c, st, col0, row0);
          else
            tma_store_2d(&map_c, st, col0, row0);
          bulk_commit();
        }
        stage_buf ^= 1;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // smem reads of the stores done (writes complete with the grid)
  }
  tc_fence_before();
  cluster_sync();  // the peer's epilogue arrivals and the leader's MMAs are done before TMEM is released
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
  }
}

// split-K finalize: out (op)= sum_s ws[s][M][N] in fixed split order (deterministic, no atomics).
// mode: EPI_BF16 / EPI_BF16_GELU -> bf16 store, EPI_F32 -> fp32 store, EPI_F32_ADD -> fp32 +=.
// Four columns per thread (N % 4 == 0, the common case) with 32-bit index math.
template <bool VEC4>
__global__ void gemm_finalize(const float* __restrict__ ws, int splits, int M, int N, void* __restrict__ out, int ldo,
                              int mode) {
  pdl_wait();
  pdl_trigger();
  const int W = VEC4 ? N / 4 : N;
  const int total = M * W;
  const size_t slab = (size_t)M * N;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int r = i / W, c = (i - r * W) * (VEC4 ? 4 : 1);
    const size_t src = (size_t)r * N + c;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    for (int sp = 0; sp < splits; ++sp) {
      if (VEC4) {
        const float4 w = *reinterpret_cast<const float4*>(ws + sp * slab + src);
        v[0] += w.x; v[1] += w.y; v[2] += w.z; v[3] += w.w;
      } else {
        v[0] += ws[sp * slab + src];
      }
    }
    const size_t dst = (size_t)r * ldo + c;
#pragma unroll
    for (int j = 0; j < (VEC4 ? 4 : 1); ++j) {
      float x = v[j];
      if (mode == EPI_BF16_GELU) x = gelu_tanh_fast(x);
      if (mode == EPI_BF16 || mode == EPI_BF16_GELU) reinterpret_cast<__nv_bfloat16*>(out)[dst + j] = __float2bfloat16(x);
      else if (mode == EPI_F32) reinterpret_cast<float*>(out)[dst + j] = x;
      else reinterpret_cast<float*>(out)[dst + j] += x;
    }
  }
}

// ------------------------------------------------------------------ host side
static int make_map(MaceCtx* ctx, CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                    uint32_t box_inner, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ctx->encode_tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

// output map of the TMA-store epilogue: {cols, rows} (or {cols, rows, splits} for split-K slabs),
// box = {128 bytes of columns, 32 rows}, 128B swizzle (matches stage_row_chunk16)
static int make_map_c(MaceCtx* ctx, CUtensorMap* map, const GemmEpilogue& ep, int M, int N, int splits) {
  const bool bf16 = ep.mode == EPI_BF16 || ep.mode == EPI_BF16_GELU || ep.mode == EPI_BF16_SWIGLU;
  const uint64_t es = bf16 ? 2 : 4;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)splits};
  cuuint64_t strides[2] = {(cuuint64_t)ep.ldo * es, (cuuint64_t)ep.split_stride * es};
  cuuint32_t box[3] = {(cuuint32_t)(128 / es), 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const int rank = ep.split_stride ? 3 : 2;
  CUresult r = ctx->encode_tiled(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank,
                                 ep.out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

// the TMA-store epilogue needs 16-byte aligned output rows (and slabs)
static bool tma_epi_ok(const GemmEpilogue& ep) {
  const size_t es = (ep.mode == EPI_BF16 || ep.mode == EPI_BF16_GELU || ep.mode == EPI_BF16_SWIGLU) ? 2 : 4;
  return ((uintptr_t)ep.out & 15) == 0 && ((size_t)ep.ldo * es) % 16 == 0 && (ep.split_stride * es) % 16 == 0;
}

template <int BN, bool A_MN, bool B_MN, bool TMA_EPI>
static int launch_gemm(MaceCtx* ctx, const MaceGemmArgs* g, int splits, cudaStream_t stream, const GemmEpilogue& ep) {
  using Cfg = GemmCfg<BN>;
  CUtensorMap ma, mb, mc;
  // A logical [M,K]; K-major storage [M, lda>=K], MN-major storage [K, lda>=M]
  int rc = A_MN ? make_map(ctx, &ma, g->a, g->M, g->K, g->lda, 64, kBK) : make_map(ctx, &ma, g->a, g->K, g->M, g->lda, kBK, kBM);
  if (rc) return mace_fail(ctx, MACE_ERR_LAUNCH, "gemm: tensor map A encode failed");
  const bool swiglu = ep.mode == EPI_BF16_SWIGLU;
  rc = B_MN ? make_map(ctx, &mb, g->b, g->N, g->K, g->ldb, 64, kBK)
            : make_map(ctx, &mb, g->b, g->K, swiglu ? 2 * g->N : g->N, g->ldb, kBK, swiglu ? BN / 2 : BN);
  if (rc) return mace_fail(ctx, MACE_ERR_LAUNCH, "gemm: tensor map B encode failed");
  GemmParams p;
  p.M = g->M;
  p.N = g->N;
  p.K = g->K;
  p.swiglu = swiglu ? 1 : 0;
  p.num_m = (g->M + kBM - 1) / kBM;
  p.num_n = swiglu ? (g->N + BN / 2 - 1) / (BN / 2) : (g->N + BN - 1) / BN;
  p.kb_total = (g->K + kBK - 1) / kBK;
  p.kb_per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  p.ep = ep;
  p.c_slab = ep.split_stride != 0;
  p.c_reduce = ep.mode == EPI_F32_ADD || ep.mode == EPI_F32_ATOMIC;
  p.b_static = (g->flags & MACE_GEMM_B_STATIC) ? 1 : 0;
#ifdef MACE_GEMM_TRACE
  p.dbg = g_gemm_dbg_host;
#else
  p.dbg = 0;
#endif
  if (TMA_EPI) {
    if (make_map_c(ctx, &mc, ep, g->M, g->N, p.c_slab ? p.splits : 1))
      return mace_fail(ctx, MACE_ERR_LAUNCH, "gemm: tensor map C encode failed");
  } else {
    mc = ma;  // unused
  }
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, TMA_EPI>;
  static bool attr_set = false;  // per-instantiation; attribute is process-wide and idempotent
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    attr_set = true;
  }
  // ring depth: never more stages than k-blocks per split; MACE_GEMM_STAGES caps it (sweeps)
  static const int stage_cap = [] {
    const char* e = getenv("MACE_GEMM_STAGES");
    return e ? atoi(e) : 0;
  }();
  int stages = Cfg::kStages;
  if (stages > p.kb_per_split) stages = p.kb_per_split;
  if (stage_cap > 0 && stages > stage_cap) stages = stage_cap;
  if (stages < 2) stages = 2;
  p.stages = stages;
  const int smem_bytes = stages * Cfg::kStageBytes + Cfg::kCBytes + 1024 + 256;
  const int tiles = p.num_m * p.num_n * p.splits;
  const int grid = tiles < ctx->num_sms ? tiles : ctx->num_sms;
  launch_k(kern, grid, 256, smem_bytes, stream, ma, mb, mc, p);
  ctx->launches++;
  return 0;
}

template <int BN, bool A_MN, bool B_MN>
static int launch_gemm2(MaceCtx* ctx, const MaceGemmArgs* g, cudaStream_t stream, const GemmEpilogue& ep) {
  using Cfg = Gemm2Cfg<BN>;
  CUtensorMap ma, mb, mc;
  if (A_MN ? make_map(ctx, &ma, g->a, g->M, g->K, g->lda, 64, kBK) : make_map(ctx, &ma, g->a, g->K, g->M, g->lda, kBK, 128))
    return mace_fail(ctx, MACE_ERR_LAUNCH, "gemm2: tensor map A encode failed");
  const bool swiglu = ep.mode == EPI_BF16_SWIGLU;
  if (B_MN ? make_map(ctx, &mb, g->b, g->N, g->K, g->ldb, 64, kBK)
           : make_map(ctx, &mb, g->b, g->K, swiglu ? 2 * g->N : g->N, g->ldb, kBK, BN / 2))
    return mace_fail(ctx, MACE_ERR_LAUNCH, "gemm2: tensor map B encode failed");
  GemmParams p{};
  p.M = g->M;
  p.N = g->N;
  p.K = g->K;
  p.swiglu = swiglu ? 1 : 0;
  p.num_m = (g->M + 255) / 256;
  p.num_n = swiglu ? (g->N + BN / 2 - 1) / (BN / 2) : (g->N + BN - 1) / BN;
  p.kb_total = (g->K + kBK - 1) / kBK;
  p.kb_per_split = p.kb_total;
  p.splits = 1;
  p.ep = ep;
  p.c_slab = 0;
  p.c_reduce = ep.mode == EPI_F32_ADD || ep.mode == EPI_F32_ATOMIC;
  p.b_static = (g->flags & MACE_GEMM_B_STATIC) ? 1 : 0;
  p.dbg = 0;
  if (ep.mode == EPI_ARGMAX)
    mc = ma;  // unused: the argmax epilogue publishes keys with atomics
  else if (make_map_c(ctx, &mc, ep, g->M, g->N, 1))
    return mace_fail(ctx, MACE_ERR_LAUNCH, "gemm2: tensor map C encode failed");
  auto kern = gemm_tc2_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    attr_set = true;
  }
  const int tiles = p.num_m * p.num_n;
  const int pairs = ctx->num_sms / 2;
  const int grid = 2 * (tiles < pairs ? tiles : pairs);
  launch_k(kern, grid, 256, Cfg::kSmemBytes, stream, ma, mb, mc, p);
  ctx->launches++;
  return 0;
}

template <int BN>
static int dispatch_pair(MaceCtx* ctx, const MaceGemmArgs* g, cudaStream_t s, const GemmEpilogue& ep) {
  if (!g->a_mn_major && !g->b_mn_major) return launch_gemm2<BN, false, false>(ctx, g, s, ep);
  if (!g->a_mn_major && g->b_mn_major) return launch_gemm2<BN, false, true>(ctx, g, s, ep);
  if (g->a_mn_major && !g->b_mn_major) return launch_gemm2<BN, true, false>(ctx, g, s, ep);
  return launch_gemm2<BN, true, true>(ctx, g, s, ep);
}

template <int BN, bool T>
static int dispatch_major_t(MaceCtx* ctx, const MaceGemmArgs* g, int splits, cudaStream_t s, const GemmEpilogue& ep) {
  if (!g->a_mn_major && !g->b_mn_major) return launch_gemm<BN, false, false, T>(ctx, g, splits, s, ep);
  if (!g->a_mn_major && g->b_mn_major) return launch_gemm<BN, false, true, T>(ctx, g, splits, s, ep);
  if (g->a_mn_major && !g->b_mn_major) return launch_gemm<BN, true, false, T>(ctx, g, splits, s, ep);
  return launch_gemm<BN, true, true, T>(ctx, g, splits, s, ep);
}

template <int BN>
static int dispatch_major(MaceCtx* ctx, const MaceGemmArgs* g, int splits, cudaStream_t s, const GemmEpilogue& ep) {
  static const bool no_tma_epi = getenv("MACE_GEMM_NO_TMA_EPI") != nullptr;  // A/B comparisons only
  if (ep.mode != EPI_ARGMAX && tma_epi_ok(ep) && !no_tma_epi) return dispatch_major_t<BN, true>(ctx, g, splits, s, ep);
  return dispatch_major_t<BN, false>(ctx, g, splits, s, ep);
}

}  // namespace mace

using namespace mace;

#ifdef MACE_GEMM_TRACE
extern "C" int mace_debug_gemm_trace(void* buf, int dbg) {
  g_gemm_dbg_host = dbg;
  return cudaMemcpyToSymbol(g_gemm_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int mace_gemm_bf16(mace_ctx* ctx_, const MaceGemmArgs* g, void* stream_) {
  MaceCtx* ctx = ctx_;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  if (!ctx || !g) return MACE_ERR_ARG;
  if (g->M <= 0 || g->N <= 0 || g->K <= 0) return 0;  // empty ragged batch: nothing to do
  if ((g->lda & 7) || (g->ldb & 7) || ((uintptr_t)g->a & 15) || ((uintptr_t)g->b & 15))
    return mace_fail(ctx, MACE_ERR_ARG, "gemm: operands need 16-byte aligned rows (ld % 8 == 0)");
  if (g->mode < EPI_BF16 || g->mode > EPI_ARGMAX) return mace_fail(ctx, MACE_ERR_ARG, "gemm: bad epilogue mode");
  const bool argmax = g->mode == EPI_ARGMAX;
  if (argmax && (g->bias || g->split_k > 1 || ((uintptr_t)g->out & 7)))
    return mace_fail(ctx, MACE_ERR_ARG, "gemm: the argmax epilogue takes 8-byte aligned keys, no bias, no split-K");
  const bool swiglu = g->mode == EPI_BF16_SWIGLU;
  if (swiglu && (g->a_mn_major || g->b_mn_major || g->bias || g->split_k > 1))
    return mace_fail(ctx, MACE_ERR_UNSUPPORTED, "gemm: SwiGLU epilogue needs K-major operands, no bias, no split-K");

  // tile shape (tools/gemm_sweep.py on B200). Big GEMMs (>= one full wave of 256 x 256 pair tiles): the
  // CTA-pair kernel (MN-major operands: single-CTA BN 256). Otherwise a per-k-block cost model fitted on the
  // tick's shapes picks among single-CTA BN 64 / 128 / 192 / 256 and pair BN 128:
  //   t ~ waves x k-blocks x c(BN),  c = 0.17 / 0.19 / 0.34 / 0.49 us (single), 0.155 us (pair 128)
  // (a fixed ~4 us launch / fill / epilogue cost is common to all, the pair kernel pays ~0.6 us more and is
  // considered from 32 k-blocks). Split-K only
  // for < 37 tiles with >= 24
  // k-blocks per split: measured slower everywhere else (slab round trip + finalize launch).
  const int num_m = (g->M + kBM - 1) / kBM;
  const int num_m2 = (g->M + 255) / 256;
  const int kb_total = (g->K + kBK - 1) / kBK;
  const bool pair_ok = g->split_k <= 0 && g->mode != EPI_F32_ATOMIC &&
                       (argmax || (((uintptr_t)g->out & 15) == 0 &&
                        ((size_t)g->ldo * ((g->mode == EPI_BF16 || g->mode == EPI_BF16_GELU || swiglu) ? 2 : 4)) % 16 == 0));
  const long sms = ctx->num_sms, pairs = ctx->num_sms / 2;
  int bn = 128, pair_bn = 0;
  if (swiglu) {  // 256-wide accumulator tiles = 128 gate + 128 up columns of the same 128 outputs
    if (!pair_ok) return mace_fail(ctx, MACE_ERR_ARG, "gemm: SwiGLU output needs 16-byte aligned rows");
    bn = 256;
    // pair tiles from one wave on, and for decode-sized M (one 256-row pair tile holds all rows: same CTA count
    // as two single-CTA m-tiles, half the weight bytes per SM)
    if ((long)num_m2 * ((g->N + 127) / 128) >= sms || (num_m2 == 1 && g->M > 128)) pair_bn = 256;
  } else if (pair_ok && (long)num_m2 * ((g->N + 255) / 256) >= sms) {
    pair_bn = 256;
  } else if (!pair_ok && (long)num_m * ((g->N + 255) / 256) >= sms) {
    bn = 256;
  } else {
    static const int kBn[4] = {64, 128, 192, 256};
    static const double kCost[4] = {0.17, 0.19, 0.34, 0.49};
    double best = 1e30;
    for (int c = 0; c < 4; ++c) {
      const long t = (long)num_m * ((g->N + kBn[c] - 1) / kBn[c]);
      const double cost = (double)((t + sms - 1) / sms) * kb_total * kCost[c];
      if (cost < best) {
        best = cost;
        bn = kBn[c];
      }
    }
    if (pair_ok && kb_total >= 32) {  // the pair kernel's longer fill (~0.6 us) only pays off over long K loops
      const long t2 = (long)num_m2 * ((g->N + 127) / 128);
      const double c128 = (double)((t2 + pairs - 1) / pairs) * kb_total * 0.155 + 0.6;
      if (c128 < best) {
        pair_bn = 128;
        best = c128;
      }
      // pair BN 64 (each CTA stages 32 weight rows per k-block): sub-wave M <= ~1.2k projections with long K, e.g.
      // M=256 N=2048 K=2048 9.4 -> 8.2 us, M=600 N=768 K=3072 11.9 -> 10.3 us (profiles/r2s5_pair64_sweep.log);
      // K-major B only (the MN-major B loader moves 64-wide blocks of BN/2 >= 64 columns)
      if (!g->b_mn_major && g->M > 128) {  // M <= 128 would leave the peer CTA's rows empty
        const long t64 = (long)num_m2 * ((g->N + 63) / 64);
        if ((double)((t64 + pairs - 1) / pairs) * kb_total * 0.13 + 0.6 < best) pair_bn = 64;
      }
    }
  }
  int splits = g->split_k > 0 ? g->split_k : 1;
  if (g->split_k <= 0 && !swiglu && !argmax && kb_total >= 96 && (long)num_m * ((g->N + 127) / 128) < pairs) {
    // long K over few tiles (decode-sized down projections, FT dW): split K across the idle SMs (BN 128)
    bn = 128;
    pair_bn = 0;
    const long tiles = (long)num_m * ((g->N + bn - 1) / bn);
    splits = (int)(sms / tiles);
    const int max_split = kb_total / 12;
    if (splits > max_split) splits = max_split;
    if (splits < 1) splits = 1;
  }
  // tuning override (tools/gemm_sweep.py): MACE_GEMM_FORCE="<bn>,<splits>" | "pair,<bn>" | "single"
  if (const char* f = getenv("MACE_GEMM_FORCE"); f && swiglu && !argmax) {  // SwiGLU: BN 256, pair or single only
    if (!strcmp(f, "pair,256") && pair_ok) pair_bn = 256;
    else if (!strcmp(f, "single")) pair_bn = 0;
  } else if (f && !argmax) {
    int fb = 0, fs = 0;
    if (sscanf(f, "%d,%d", &fb, &fs) == 2) {
      if (fb == 64 || fb == 128 || fb == 192 || fb == 256) bn = fb;
      if (fs >= 1) splits = fs;
      pair_bn = 0;
    } else if (sscanf(f, "pair,%d", &fb) == 1 && (fb == 64 || fb == 128 || fb == 256) && pair_ok) {
      pair_bn = fb;
    } else {
      pair_bn = 0;
    }
  }
  GemmEpilogue ep;
  ep.out = g->out;
  ep.ldo = g->ldo;
  ep.bias = reinterpret_cast<const __nv_bfloat16*>(g->bias);
  ep.alpha = g->alpha == 0.f ? 1.f : g->alpha;
  ep.mode = g->mode;
  ep.split_stride = 0;
  {
    if (pair_bn) {
      const int rc2 = pair_bn == 256   ? dispatch_pair<256>(ctx, g, stream, ep)
                      : pair_bn == 128 ? dispatch_pair<128>(ctx, g, stream, ep)
                                       : dispatch_pair<64>(ctx, g, stream, ep);
      if (rc2) return rc2;
      return mace_check_launch(ctx, "gemm2");
    }
  }
  bool need_finalize = false;
  if (splits > 1 && g->mode != EPI_F32_ATOMIC) {
    // keep the per-split slabs inside the caller's workspace
    const size_t slab = (size_t)g->M * g->N;
    const size_t fit = g->workspace ? g->workspace_bytes / (slab * 4) : 0;
    if ((size_t)splits > fit) splits = (int)fit;
    if (splits > 1) {
      const int kbp = (kb_total + splits - 1) / splits;
      splits = (kb_total + kbp - 1) / kbp;  // the splits the kernel will actually run
      ep.out = g->workspace;
      ep.ldo = g->N;
      ep.mode = EPI_F32;
      ep.split_stride = slab;
      need_finalize = true;
    } else {
      splits = 1;
    }
  }
  int rc;
  if (bn == 256)
    rc = dispatch_major<256>(ctx, g, splits, stream, ep);
  else if (bn == 192)
    rc = dispatch_major<192>(ctx, g, splits, stream, ep);
  else if (bn == 128)
    rc = dispatch_major<128>(ctx, g, splits, stream, ep);
  else
    rc = dispatch_major<64>(ctx, g, splits, stream, ep);
  if (rc) return rc;
  if (need_finalize) {
    const bool vec4 = (g->N % 4) == 0;
    const long long work = (long long)g->M * (vec4 ? g->N / 4 : g->N);
    int fgrid = (int)((work + 255) / 256);
    if (fgrid > ctx->num_sms * 8) fgrid = ctx->num_sms * 8;
    if (vec4)
      launch_k(gemm_finalize<true>, fgrid, 256, 0, stream, reinterpret_cast<const float*>(g->workspace), splits, g->M,
               g->N, g->out, g->ldo, g->mode);
    else
      launch_k(gemm_finalize<false>, fgrid, 256, 0, stream, reinterpret_cast<const float*>(g->workspace), splits, g->M,
               g->N, g->out, g->ldo, g->mode);
    ctx->launches++;
  }
  return mace_check_launch(ctx, "gemm");
}
