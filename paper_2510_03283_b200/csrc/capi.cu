// Context lifecycle, error convention and driver-entry-point plumbing for the C-ABI.
#include <cstdio>

#include "common.cuh"
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

mace::HostProf mace::g_host_prof;
static PFN_cuTensorMapEncodeTiled_v12000 g_encode_real = nullptr;
static CUresult CUDAAPI encode_timed(CUtensorMap* m, CUtensorMapDataType t, cuuint32_t r, void* p, const cuuint64_t* d,
                                     const cuuint64_t* st, const cuuint32_t* b, const cuuint32_t* e,
                                     CUtensorMapInterleave il, CUtensorMapSwizzle sw, CUtensorMapL2promotion l2,
                                     CUtensorMapFloatOOBfill f) {
  const auto t0 = std::chrono::steady_clock::now();
  const CUresult res = g_encode_real(m, t, r, p, d, st, b, e, il, sw, l2, f);
  mace::g_host_prof.encode_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  mace::g_host_prof.n_encode++;
  return res;
}

using namespace mace;

// [launch seconds, launches, encode seconds, encodes] since the last call (MACE_HOST_PROF=1 only)
extern "C" int mace_debug_host_prof(double* out) {
  out[0] = g_host_prof.launch_s;
  out[1] = (double)g_host_prof.n_launch;
  out[2] = g_host_prof.encode_s;
  out[3] = (double)g_host_prof.n_encode;
  g_host_prof = HostProf();
  return host_prof_on() ? 0 : -1;
}

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
  if (host_prof_on()) {
    g_encode_real = ctx->encode_tiled;
    ctx->encode_tiled = encode_timed;
  }
  *out = ctx;
  return MACE_OK;
}

extern "C" int mace_ctx_destroy(mace_ctx* ctx) {
  delete ctx;
  return MACE_OK;
}

extern "C" const char* mace_last_error(mace_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null ctx"; }

extern "C" long long mace_launch_count(mace_ctx* ctx) { return ctx ? ctx->launches : 0; }
