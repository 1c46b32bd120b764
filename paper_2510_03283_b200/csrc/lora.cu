// Per-tenant LoRA adapters on the selected layers (the paper's per-user adapter phi_u,
// PAPER.md:440-441, over the reference's multi-tenant environments, config.py:212-239).
//
// All tenants' adapters of a projection are stacked: A_all [R, in], B^T_all [R, out] with R = tenants x rank.
// For a ragged batch whose rows belong to different tenants:
//   Z  = X A_all^T                       one bf16 tcgen05 GEMM (N = R: every tenant's shrink at once)
//   Zm = mask(Z)                         this kernel: keep the row's own tenant block, scaled by alpha / rank
//   qkv, up:  [X | Zm] [W | B_all]^T     the base GEMM with K extended by R (the augmented weight), so the
//                                        fused bias / GELU / SwiGLU epilogues see base + adapter
//   o, down:  x += Zm B^T_all            a second GEMM into the fp32 residual (K = R)
// The wasted columns of other tenants cost R / in of the base GEMM (<= 3% at 8 tenants x rank 16, d 4096),
// against gathering rows per tenant (extra copies, per-tenant launches).
#include "common.cuh"
#include "mace_internal.h"

namespace mace {

__global__ void lora_mask_kernel(const float* __restrict__ z, int ldz, const int* __restrict__ tenant, int n, int rank,
                                 int R, float scale, __nv_bfloat16* __restrict__ out, int ldo) {
  pdl_wait();
  pdl_trigger();
  const int per = R / 8;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)n * per) return;
  const int row = (int)(i / per), c = (int)(i % per) * 8;
  const int t = tenant ? tenant[row] : -1;
  float y[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) y[j] = 0.f;
  if (t >= 0) {
    const float4* zp = reinterpret_cast<const float4*>(z + (size_t)row * ldz + c);
    const float4 a = zp[0], b = zp[1];
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if ((c + j) / rank == t) y[j] = scale * v[j];
  }
  *reinterpret_cast<uint4*>(out + (size_t)row * ldo + c) =
      make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]), pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7]));
}

// fp32 [n, cols] (ld ldx) -> bf16 (ld ldy), 8 columns per thread: the backward's dY of a LoRA layer lands in the
// first cols of a [n, cols + R] buffer whose last R columns take the masked dZ ([dY | dZ] . [W; A] is one GEMM)
__global__ void f32_to_bf16_2d_kernel(const float* __restrict__ x, int ldx, int n, int cols,
                                      __nv_bfloat16* __restrict__ y, int ldy) {
  pdl_wait();
  pdl_trigger();
  const int per = cols / 8;
  const long long total = (long long)n * per;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / per), c = (int)(i % per) * 8;
    const float4* xp = reinterpret_cast<const float4*>(x + (size_t)row * ldx + c);
    const float4 a = xp[0], b = xp[1];
    *reinterpret_cast<uint4*>(y + (size_t)row * ldy + c) =
        make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
  }
}

// B^T rows of the adapters [rows, out] (bf16, the AdamW working copy) -> columns [col0, col0 + rows) of the
// augmented base weight [out, ldd] ([W | B], K-major for the forward GEMM). One thread per (out row, col).
__global__ void lora_bt_scatter_kernel(const __nv_bfloat16* __restrict__ bt, int rows, int out,
                                       __nv_bfloat16* __restrict__ dst, int ldd, int col0) {
  pdl_wait();
  pdl_trigger();
  const long long total = (long long)out * rows;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int o = (int)(i / rows), j = (int)(i % rows);
    dst[(size_t)o * ldd + col0 + j] = bt[(size_t)j * out + o];
  }
}

}  // namespace mace

using namespace mace;

extern "C" int mace_f32_to_bf16_2d(mace_ctx* ctx, const float* x, int ldx, int n, int cols, void* y, int ldy,
                                   void* stream) {
  if (n <= 0 || cols <= 0) return 0;
  if (cols % 8 || ldx % 4 || ldy % 8) return mace_fail(ctx, MACE_ERR_ARG, "f32_to_bf16_2d: cols % 8, ldx % 4, ldy % 8");
  const long long work = (long long)n * (cols / 8);
  long long grid = (work + 255) / 256;
  if (grid > (long long)ctx->num_sms * 16) grid = ctx->num_sms * 16;
  launch_k(f32_to_bf16_2d_kernel, (int)grid, 256, 0, (cudaStream_t)stream, x, ldx, n, cols, (__nv_bfloat16*)y, ldy);
  ctx->launches++;
  return mace_check_launch(ctx, "f32_to_bf16_2d");
}

extern "C" int mace_lora_bt_scatter(mace_ctx* ctx, const void* bt, int rows, int out, void* dst, int ldd, int col0,
                                    void* stream) {
  if (rows <= 0 || out <= 0) return 0;
  const long long work = (long long)rows * out;
  long long grid = (work + 255) / 256;
  if (grid > (long long)ctx->num_sms * 16) grid = ctx->num_sms * 16;
  launch_k(lora_bt_scatter_kernel, (int)grid, 256, 0, (cudaStream_t)stream, (const __nv_bfloat16*)bt, rows, out,
           (__nv_bfloat16*)dst, ldd, col0);
  ctx->launches++;
  return mace_check_launch(ctx, "lora_bt_scatter");
}

extern "C" int mace_lora_mask(mace_ctx* ctx, const float* z, int ldz, const int* tenant, int n, int rank, int R,
                              float scale, void* out, int ldo, void* stream) {
  if (n <= 0) return 0;
  if (R % 8 || rank <= 0 || ldz % 4 || ldo % 8) return mace_fail(ctx, MACE_ERR_ARG, "lora_mask: R % 8, ldz % 4, ldo % 8");
  const long long work = (long long)n * (R / 8);
  launch_k(lora_mask_kernel, (int)((work + 255) / 256), 256, 0, (cudaStream_t)stream, z, ldz, tenant, n, rank, R, scale,
           (__nv_bfloat16*)out, ldo);
  ctx->launches++;
  return mace_check_launch(ctx, "lora_mask");
}
