// (4) KV page allocate / evict / compaction for the colocated memory manager.
//
// The reference keeps KV as MB arithmetic: decode growth engine.py:512-514, per-head prune trim
// engine.py:506-529 (kept[h] -> caps[h], oldest slots first), prefix-cache insert/evict
// cache.py:186-238. Here the same decisions move real pages:
//   decode_alloc  before a tick: every decode row appends slot j = dec_end; a head whose ring is full
//                 pops a page from the device free stack (no host round trip)
//   trim          after a tick: the reference's post-tick kept[h] sets dec_first = dec_end - kept[h];
//                 ring pages entirely below dec_first are pushed back and the ring is compacted
//   release       a retiring request returns all its decode pages
//   compact       re-base a head's ring at its retained window: the window [dec_first, dec_end) shifts down to
//                 ring offset 0 inside the same pages, so a window that straddled a page boundary it does not
//                 need (e.g. 4 tokens over 2 pages after a prune trim) frees its now-empty last page
//   page_copy     copy-on-diverge of a partially shared prompt page (trie split at a non page-aligned
//                 token, cache.py:79-105) across every layer of both pools
// Pops and pushes never run in the same kernel, so the stack needs no ABA protection.
// free_top points at int[2] = {stack top, status}; status bit 0 = a pop found the stack empty (the row was
// pointed at kv.sink_page, a reserved page outside the stack). The host mirror makes that unreachable.
#include "common.cuh"
#include "mace_internal.h"

namespace mace {

__global__ void decode_alloc_kernel(const int* __restrict__ slots, int n, MaceKvLayout kv) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int H = kv.n_kv_heads;
  if (i >= n * H) return;
  const int slot = slots[i / H], h = i % H;
  const int kvh = slot * H + h;
  const int j = kv.dec_end[slot];  // slot index being appended (dec_end bumped after all heads)
  const int rel = j - kv.dec_base[kvh];
  if (rel % kPageTokens == 0) {
    const int top = atomicSub(kv.free_top, 1) - 1;
    int page;
    if (top >= 0) {
      page = kv.free_stack[top];
    } else {
      // pool exhausted: unreachable when the host mirror (kvmanager.DecodePageMirror) admitted the tick.
      // Defence in depth: undo the pop, point the row at the reserved sink page (writes and reads stay in
      // bounds) and raise the status word the host reads with mace_kv_status.
      atomicAdd(kv.free_top, 1);
      atomicOr(kv.free_top + 1, 1);
      page = kv.sink_page;
    }
    kv.dtab[(size_t)kvh * kv.max_dec_pages + rel / kPageTokens] = page;
  }
}

__global__ void bump_end_kernel(const int* __restrict__ slots, int n, int* __restrict__ dec_end) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dec_end[slots[i]] += 1;
}

// kept: [n][H] post-tick retained decode slots per head (Engine._exec_decode's rs.kept)
__global__ void trim_kernel(const int* __restrict__ slots, const int* __restrict__ kept, int n, MaceKvLayout kv) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int H = kv.n_kv_heads;
  if (i >= n * H) return;
  const int slot = slots[i / H], h = i % H;
  const int kvh = slot * H + h;
  const int de = kv.dec_end[slot];
  const int first = max(kv.dec_first[kvh], de - kept[i]);
  kv.dec_first[kvh] = first;
  int base = kv.dec_base[kvh];
  int* ring = kv.dtab + (size_t)kvh * kv.max_dec_pages;
  int drop = 0;
  while (first - base >= kPageTokens) {
    if (ring[drop] != kv.sink_page) kv.free_stack[atomicAdd(kv.free_top, 1)] = ring[drop];
    ++drop;
    base += kPageTokens;
  }
  if (drop) {
    const int live = (de - 1 - kv.dec_base[kvh]) / kPageTokens + 1;
    for (int r = 0; r + drop < live; ++r) ring[r] = ring[r + drop];
    kv.dec_base[kvh] = base;
  }
}

__global__ void release_kernel(const int* __restrict__ slots, int n, MaceKvLayout kv) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int H = kv.n_kv_heads;
  if (i >= n * H) return;
  const int slot = slots[i / H], h = i % H;
  const int kvh = slot * H + h;
  const int de = kv.dec_end[slot], base = kv.dec_base[kvh];
  const int live = de > base ? (de - 1 - base) / kPageTokens + 1 : 0;
  const int* ring = kv.dtab + (size_t)kvh * kv.max_dec_pages;
  for (int r = 0; r < live; ++r)
    if (ring[r] != kv.sink_page) kv.free_stack[atomicAdd(kv.free_top, 1)] = ring[r];
  kv.dec_base[kvh] = 0;
  kv.dec_first[kvh] = 0;
}

// items int2 [n] = (slot, head), chosen by the host mirror (DecodePageMirror.compact_candidates): windows of at most
// max_w tokens that one page fewer can hold. grid (n, L, 2 pools): the CTA stages the window's rows of one layer
// and pool in shared memory (every read before any write: source and destination overlap), then writes them
// back at ring offsets 0..w-1. dec_base / the free stack change only in the commit kernel after it.
__global__ void kv_compact_move_kernel(const int2* __restrict__ items, MaceKvLayout kv, int hd,
                                       long long pages_per_layer, __nv_bfloat16* __restrict__ kp,
                                       __nv_bfloat16* __restrict__ vp) {
  extern __shared__ uint4 stage[];
  pdl_wait();
  pdl_trigger();
  const int2 it = items[blockIdx.x];
  const int H = kv.n_kv_heads, kvh = it.x * H + it.y;
  const int f = kv.dec_first[kvh], b = kv.dec_base[kvh], w = kv.dec_end[it.x] - f;
  const int* ring = kv.dtab + (size_t)kvh * kv.max_dec_pages;
  __nv_bfloat16* pool = (blockIdx.z ? vp : kp) + (size_t)blockIdx.y * pages_per_layer * kPageTokens * hd;
  const int cpr = hd / 8;  // 16-byte chunks per token row
  for (int i = threadIdx.x; i < w * cpr; i += blockDim.x) {
    const int off = f - b + i / cpr;
    stage[i] = *reinterpret_cast<const uint4*>(
        pool + ((size_t)ring[off / kPageTokens] * kPageTokens + off % kPageTokens) * hd + (i % cpr) * 8);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < w * cpr; i += blockDim.x) {
    const int off = i / cpr;
    *reinterpret_cast<uint4*>(pool + ((size_t)ring[off / kPageTokens] * kPageTokens + off % kPageTokens) * hd +
                              (i % cpr) * 8) = stage[i];
  }
}

__global__ void kv_compact_commit_kernel(const int2* __restrict__ items, int n, MaceKvLayout kv) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int2 it = items[i];
  const int kvh = it.x * kv.n_kv_heads + it.y;
  const int f = kv.dec_first[kvh], b = kv.dec_base[kvh], e = kv.dec_end[it.x];
  const int old_pages = (e - 1 - b) / kPageTokens + 1, new_pages = (e - 1 - f) / kPageTokens + 1;
  const int* ring = kv.dtab + (size_t)kvh * kv.max_dec_pages;
  for (int r = new_pages; r < old_pages; ++r)
    if (ring[r] != kv.sink_page) kv.free_stack[atomicAdd(kv.free_top, 1)] = ring[r];
  kv.dec_base[kvh] = f;
}

__global__ void reset_slot_kernel(const int* __restrict__ slots, int n, MaceKvLayout kv) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) kv.dec_end[slots[i]] = 0;
}

// copies[n][4] = (src_group, dst_group, n_tokens, 0): rows [0, n_tokens) of every head page of the
// group, every layer, both pools. pool layout [L][pages][16][hd].
__global__ void page_copy_kernel(const int4* __restrict__ copies, int n, int H, int hd, long long pages_per_layer,
                                 int L, __nv_bfloat16* __restrict__ kp, __nv_bfloat16* __restrict__ vp) {
  pdl_wait();
  pdl_trigger();
  const int4 c = copies[blockIdx.x];
  const int row_elems = c.z * hd;
  for (int l = 0; l < L; ++l) {
    for (int h = 0; h < H; ++h) {
      const size_t src = ((size_t)l * pages_per_layer + (size_t)c.x * H + h) * kPageTokens * hd;
      const size_t dst = ((size_t)l * pages_per_layer + (size_t)c.y * H + h) * kPageTokens * hd;
      for (int e = threadIdx.x * 8; e < row_elems; e += blockDim.x * 8) {
        *reinterpret_cast<uint4*>(kp + dst + e) = *reinterpret_cast<const uint4*>(kp + src + e);
        *reinterpret_cast<uint4*>(vp + dst + e) = *reinterpret_cast<const uint4*>(vp + src + e);
      }
    }
  }
}

}  // namespace mace

using namespace mace;

extern "C" int mace_kv_decode_alloc(mace_ctx* ctx, const MaceKvLayout* kv, const int* slots, int n, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int tot = n * kv->n_kv_heads;
  launch_k(decode_alloc_kernel, (tot + 255) / 256, 256, 0, s, slots, n, *kv);
  launch_k(bump_end_kernel, (n + 255) / 256, 256, 0, s, slots, n, kv->dec_end);
  ctx->launches += 2;
  return mace_check_launch(ctx, "kv_decode_alloc");
}

extern "C" int mace_kv_trim(mace_ctx* ctx, const MaceKvLayout* kv, const int* slots, const int* kept, int n,
                            void* stream) {
  if (n <= 0) return 0;
  const int tot = n * kv->n_kv_heads;
  launch_k(trim_kernel, (tot + 255) / 256, 256, 0, (cudaStream_t)stream, slots, kept, n, *kv);
  ctx->launches++;
  return mace_check_launch(ctx, "kv_trim");
}

extern "C" int mace_kv_release(mace_ctx* ctx, const MaceKvLayout* kv, const int* slots, int n, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int tot = n * kv->n_kv_heads;
  launch_k(release_kernel, (tot + 255) / 256, 256, 0, s, slots, n, *kv);
  launch_k(reset_slot_kernel, (n + 255) / 256, 256, 0, s, slots, n, *kv);
  ctx->launches += 2;
  return mace_check_launch(ctx, "kv_release");
}

extern "C" int mace_kv_page_copy(mace_ctx* ctx, const int* copies, int n, int n_kv_heads, int hd, long long pages_per_layer,
                                 int n_layers, void* k_pools, void* v_pools, void* stream) {
  if (n <= 0) return 0;
  launch_k(page_copy_kernel, n, 128, 0, (cudaStream_t)stream, reinterpret_cast<const int4*>(copies), n, n_kv_heads, hd,
                                                        pages_per_layer, n_layers, (__nv_bfloat16*)k_pools,
                                                        (__nv_bfloat16*)v_pools);
  ctx->launches++;
  return mace_check_launch(ctx, "kv_page_copy");
}

namespace mace {
__global__ void set_tables_kernel(const int* __restrict__ slots, const int* __restrict__ tables, int n, int ncols,
                                  int* __restrict__ ptab, int maxpp) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (r >= n) return;
  for (int c = threadIdx.x; c < ncols && c < maxpp; c += blockDim.x)
    ptab[(size_t)slots[r] * maxpp + c] = tables[(size_t)r * ncols + c];
}
__global__ void scatter_tokens_kernel(const int* __restrict__ src, const int* __restrict__ slots, int n,
                                      int* __restrict__ last_token) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) last_token[slots[i]] = src[i];
}
}  // namespace mace

extern "C" int mace_kv_set_prompt_tables(mace_ctx* ctx, const MaceKvLayout* kv, const int* slots, const int* tables,
                                         int n, int ncols, void* stream) {
  if (n <= 0) return 0;
  launch_k(mace::set_tables_kernel, n, 128, 0, (cudaStream_t)stream, slots, tables, n, ncols, const_cast<int*>(kv->ptab),
                                                               kv->max_prompt_pages);
  ctx->launches++;
  return mace::mace_check_launch(ctx, "kv_set_prompt_tables");
}

extern "C" int mace_scatter_tokens(mace_ctx* ctx, const int* src, const int* slots, int n, int* last_token,
                                   void* stream) {
  if (n <= 0) return 0;
  launch_k(mace::scatter_tokens_kernel, (n + 255) / 256, 256, 0, (cudaStream_t)stream, src, slots, n, last_token);
  ctx->launches++;
  return mace::mace_check_launch(ctx, "scatter_tokens");
}

extern "C" int mace_kv_status(mace_ctx* ctx, const MaceKvLayout* kv, int* out2) {
  if (!ctx || !kv || !out2) return MACE_ERR_ARG;
  if (cudaMemcpy(out2, kv->free_top, 2 * sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return mace_fail(ctx, MACE_ERR_CUDA, "kv_status: copy failed");
  return MACE_OK;
}

extern "C" int mace_kv_compact(mace_ctx* ctx, const MaceKvLayout* kv, const int* items, int n, int max_w, int n_layers,
                               int hd, long long pages_per_layer, void* k_pools, void* v_pools, void* stream) {
  if (n <= 0) return 0;
  if (hd % 8 || max_w <= 0 || max_w > 4 * kPageTokens)
    return mace_fail(ctx, MACE_ERR_ARG, "kv_compact: hd % 8 == 0 and 0 < max_w <= 64");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = (size_t)max_w * hd * 2;
  launch_k(kv_compact_move_kernel, dim3(n, n_layers, 2), 128, smem, s, (const int2*)items, *kv, hd, pages_per_layer,
           (__nv_bfloat16*)k_pools, (__nv_bfloat16*)v_pools);
  launch_k(kv_compact_commit_kernel, (n + 127) / 128, 128, 0, s, (const int2*)items, n, *kv);
  ctx->launches += 2;
  return mace_check_launch(ctx, "kv_compact");
}
