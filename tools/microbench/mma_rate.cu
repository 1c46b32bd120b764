// tcgen05.mma issue-rate probe: one CTA per SM, smem operands (zeros), back-to-back MMAs into TMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2510_03283_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include "common.cuh"
using namespace mace;

template <int N, int LAYOUT, int NCOMMIT, int SPIN, int RANDOM>
__global__ void __launch_bounds__(256, 1) probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bar_done, bar_ready;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (i * 2654435761u) ^ 0x9e3779b9u; h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    reinterpret_cast<uint32_t*>(smem)[i] = RANDOM ? (h & 0xBFFFBFFFu) | 0x3C003C00u : 0u;  // bf16 pairs in ~[-2, 2]
  }
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar_done, 1); mbar_init(&bar_ready, 1); mbar_arrive(&bar_ready); fence_barrier_init(); }
  fence_proxy_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, false, false);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = smem_desc(a + k * 32, 16, 1024, LAYOUT);
        uint64_t bd = smem_desc(b + k * 32, 16, 1024, LAYOUT);
        umma_bf16(tmem, ad, bd, idesc, (it | k) ? 1u : 0u);
      }
      if (NCOMMIT > 0 && (it % (NCOMMIT > 0 ? NCOMMIT : 1)) == 0) umma_commit(&bar);
      if (SPIN == 3) tc_fence_after();
      if (SPIN == 4) { mbar_wait(&bar_ready, 0); tc_fence_after(); }
    }
    long long t1 = clock64();
    umma_commit(&bar_done);
    mbar_wait(&bar_done, 0);
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  } else if (threadIdx.x >= 128) {
    // SPIN 1: 128 threads poll the completion barrier (try_wait loop), SPIN 2: one lane polls with
    // nanosleep backoff and releases the rest through a named barrier
    if (SPIN == 1) {
      mbar_wait(&bar_done, 0);
    } else if (SPIN == 2) {
      if (threadIdx.x == 128) {
        uint32_t ok = 0;
        while (!ok) {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar_done)) : "memory");
          if (!ok) __nanosleep(64);
        }
      }
      named_bar_sync(1, 128);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<256>(tmem);
}

template <int N, int LAYOUT, int NCOMMIT, int SPIN = 0, int RANDOM = 0>
void run(const char* name, int grid, int smem_kb = 80) {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  auto k = probe<N, LAYOUT, NCOMMIT, SPIN, RANDOM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
  const int iters = 2000;
  k<<<grid, 256, smem_kb * 1024>>>(d, iters);
  k<<<grid, 256, smem_kb * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-28s grid %3d: issue %6.1f cyc/MMA, complete %6.1f cyc/MMA (%s)\n", name, grid, h[0] / (4.0 * iters),
         h[1] / (4.0 * iters), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64, 2, 0>("N=64  SW128", 1);
  run<128, 2, 0>("N=128 SW128", 1);
  run<256, 2, 0>("N=256 SW128", 1);
  run<64, 2, 1>("N=64  SW128 commit/kblock", 1);
  run<256, 2, 1>("N=256 SW128 commit/kblock", 1);
  run<64, 2, 0>("N=64  SW128", 148);
  run<256, 2, 0>("N=256 SW128", 148);
  run<64, 2, 0, 0, 1>("N=64  random smem227", 1, 227);
  run<256, 2, 0, 0, 1>("N=256 random smem227", 1, 227);
  run<64, 2, 0, 0, 1>("N=64  random", 1);
  run<128, 2, 0, 0, 1>("N=128 random", 1);
  run<256, 2, 0, 0, 1>("N=256 random", 1);
  run<64, 2, 0, 0, 1>("N=64  random", 148);
  run<256, 2, 0, 0, 1>("N=256 random", 148);
  run<64, 2, 0, 3>("N=64  fence/kblock", 1);
  run<256, 2, 0, 3>("N=256 fence/kblock", 1);
  run<64, 2, 0, 4>("N=64  wait+fence/kblock", 1);
  run<256, 2, 0, 4>("N=256 wait+fence/kblock", 1);
  run<64, 2, 1, 4>("N=64  wait+fence+commit", 1);
  run<64, 2, 0, 1>("N=64  + 128 spinning", 1);
  run<256, 2, 0, 1>("N=256 + 128 spinning", 1);
  run<64, 2, 0, 2>("N=64  + 1 sleeper", 1);
  run<256, 2, 0, 2>("N=256 + 1 sleeper", 1);
  return 0;
}
