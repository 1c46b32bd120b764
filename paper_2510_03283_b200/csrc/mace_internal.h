// Internal (non-ABI) declarations shared by the .cu translation units of libmace_b200.so.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#include <unordered_map>

#include "../../include/mace_b200.h"

namespace mace {

constexpr int kPageTokens = MACE_PAGE_TOKENS;

enum EpiMode { EPI_BF16 = 0, EPI_F32 = 1, EPI_F32_ADD = 2, EPI_F32_ATOMIC = 3, EPI_BF16_GELU = 4, EPI_BF16_SWIGLU = 5, EPI_ARGMAX = 6 };

struct GemmEpilogue {
  void* out;
  int ldo;
  int mode;
  const __nv_bfloat16* bias;
  float alpha;
  size_t split_stride;  // != 0: split s writes out + s * split_stride (fp32 slabs, deterministic split-K)
};

struct MaceCtx {
  int device = 0;
  int num_sms = 148;
  long long launches = 0;
  std::string last_error;
  PFN_cuTensorMapEncodeTiled_v12000 encode_tiled = nullptr;
};

int mace_fail(MaceCtx* ctx, int code, const std::string& msg);

// tensor maps of the tensor-core prefill / FT attention (attention.cu, attention_fa2.cu)
struct TcMapsFa {
  CUtensorMap q;       // qkv [T, W], box {64, 128}: Q tiles and the dense (FT) K / V tiles
  CUtensorMap kpool;   // [pages*16, HD], box {64, 16}: one box per 16-token page
  CUtensorMap vpool;
};
int mace_check_launch(MaceCtx* ctx, const char* what);

}  // namespace mace

// opaque ABI handle is the internal struct
struct mace_ctx : public mace::MaceCtx {};
