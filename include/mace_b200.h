/*
 * mace_b200.h — C-ABI of libmace_b200.so, the sm_100a execution layer for MACE's hybrid iteration.
 *
 * The reference (macesim, a discrete-event simulator) has no native layer: every entry point below
 * replaces a cost-model *stand-in* inside the reference's hot path, named per function:
 *   Engine._execute              /root/reference/pkg/src/macesim/engine.py:573-676
 *   Engine._exec_prefill         engine.py:444-480   (prefill rows: latency = 0.5 ms/token stand-in)
 *   Engine._exec_decode          engine.py:482-532   (decode rows: 20 ms/step stand-in, KV growth + prune)
 *   Engine._exec_ft / ft_step    engine.py:534-536, alignment.py:168-172 (mu += ft_gain stand-in)
 *   dpo_loss                     alignment.py:39-47  (the scalar stage shared with the fused DPO kernel)
 *   PrefixTrie.lru_offload       cache.py:217-238    (evict decision -> page free)
 *   prune trim                   engine.py:506-529   (kept[h] trim -> page-table compaction)
 * The Python side calls these through ctypes from GpuEngine._execute (the override point the reference
 * exposes, engine.py:573); see INTEGRATION.md for the binding.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes; `stream` is a cudaStream_t passed as void*.
 *  - The caller owns ALL device memory (weights, KV pools, activations, workspaces); kernels never
 *    allocate.
 *  - Every call is stream-ordered and asynchronous; returns 0 (MACE_OK) or a negative mace_status,
 *    with a message available from mace_last_error(ctx). No exceptions cross the ABI.
 *  - No process-global mutable state: one mace_ctx per Engine / thread (threaded sweeps are safe).
 *  - There is no CPU fallback: without a B200 (sm_100) device, mace_ctx_create fails.
 */
#ifndef MACE_B200_H
#define MACE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mace_ctx mace_ctx;

enum mace_status {
  MACE_OK = 0,
  MACE_ERR_ARG = -1,
  MACE_ERR_CUDA = -2,
  MACE_ERR_LAUNCH = -3,
  MACE_ERR_NOMEM = -4,
  MACE_ERR_UNSUPPORTED = -5,
};

/* ---------------------------------------------------------------- context */
int mace_version(void);
int mace_ctx_create(int device, mace_ctx** out);
int mace_ctx_destroy(mace_ctx* ctx);
const char* mace_last_error(mace_ctx* ctx);
/* number of kernels this ctx has launched (evidence for the bench's gpu_launches) */
long long mace_launch_count(mace_ctx* ctx);

/* ---------------------------------------------------------------- (2) bf16 tcgen05 GEMM
 * C[M,N] = alpha * A[M,K] . B[N,K]^T (+bias[N]).  A is stored K-major ([M, lda]) or, with
 * a_mn_major, MN-major ([K, lda], i.e. A^T row-major); same for B.  Epilogue modes: */
enum mace_epilogue {
  MACE_EPI_BF16 = 0,       /* out bf16 = result                                  */
  MACE_EPI_F32 = 1,        /* out fp32 = result                                  */
  MACE_EPI_F32_ADD = 2,    /* out fp32 += result (residual stream, grad accumulate) */
  MACE_EPI_F32_ATOMIC = 3, /* out fp32 += result via atomics (shared destination)   */
};
typedef struct MaceGemmArgs {
  const void* a; int lda; int a_mn_major;
  const void* b; int ldb; int b_mn_major;
  int M, N, K;
  void* out; int ldo; int mode;
  const void* bias;      /* bf16 [N] or NULL (added once) */
  float alpha;           /* 0 means 1 */
  int split_k;           /* 0 = heuristic */
  void* workspace;       /* fp32 scratch for split-K with bf16 output (may be NULL) */
  size_t workspace_bytes;
} MaceGemmArgs;
int mace_gemm_bf16(mace_ctx* ctx, const MaceGemmArgs* args, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MACE_B200_H */
