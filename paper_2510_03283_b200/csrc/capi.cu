// Context lifecycle, error convention and driver-entry-point plumbing for the C-ABI.
#include <cstdio>

#include "mace_internal.h"

namespace mace {

int mace_fail(MaceCtx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return code;
}

int mace_check_launch(MaceCtx* ctx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    return mace_fail(ctx, MACE_ERR_LAUNCH, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return MACE_OK;
}

}  // namespace mace

using namespace mace;

extern "C" int mace_version(void) { return 1; }

extern "C" int mace_ctx_create(int device, mace_ctx** out) {
  if (!out) return MACE_ERR_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) {
    cudaGetLastError();
    return MACE_ERR_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return MACE_ERR_CUDA;
  if (prop.major != 10) return MACE_ERR_UNSUPPORTED;  // sm_100a kernels only: no fallback
  mace_ctx* ctx = new mace_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    delete ctx;
    return MACE_ERR_CUDA;
  }
  ctx->encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  *out = ctx;
  return MACE_OK;
}

extern "C" int mace_ctx_destroy(mace_ctx* ctx) {
  delete ctx;
  return MACE_OK;
}

extern "C" const char* mace_last_error(mace_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null ctx"; }

extern "C" long long mace_launch_count(mace_ctx* ctx) { return ctx ? ctx->launches : 0; }
