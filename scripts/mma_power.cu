// Dev probe: board power of sustained tcgen05.mma streams (every SM, ~2 s per config) for
// M = 128 vs 64, N = 64 / 128, zero vs random operands.  Run under nvidia-smi sampling.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_power mma_power.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <unistd.h>

#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"

using namespace taper;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
               : "=r"(pred));
  return pred != 0;
}

template <int M, int N>
__global__ void __launch_bounds__(128, 1) burn(long long iters, int random_ops, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  uint32_t seed = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
  for (int i = threadIdx.x; i < (48 * 1024) / 4; i += blockDim.x) {
    seed = seed * 1664525u + 1013904223u;
    reinterpret_cast<uint32_t *>(smem)[i] = random_ops ? (seed & 0xbfffbfffu) : 0u;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(M, N, false, false);
    const uint64_t a0 = umma_desc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t b0 = umma_desc_sw128(smem_u32(smem + 16384), 16, 1024);
    uint32_t phase = 0;
    for (long long it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          tc_mma_f16(tmem, a0 + uint64_t(((i & 3) * 32) >> 4), b0 + uint64_t(((i & 3) * 32) >> 4),
                     idesc, i > 0 ? 1u : 0u);
        tc_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, phase);
      phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}

template <int M, int N>
void run(int random_ops, long long *d) {
  auto k = burn<M, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  // ~2 s: 32 MMAs of max(M,128)*N/256 cycles each at ~1.8 GHz
  const long long per_iter_cycles = 32LL * 128 * N / 256;
  const long long iters = (long long)(2.0 * 1.8e9 / per_iter_cycles);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  printf("BEGIN M=%d N=%d %s\n", M, N, random_ops ? "random" : "zero");
  fflush(stdout);
  cudaEventRecord(a);
  k<<<148, 128, 50 * 1024>>>(iters, random_ops, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 148.0 * iters * 32 * 2.0 * M * N * 16;
  printf("END   M=%d N=%d %s: %.0f ms, %.1f TFLOP/s issued\n", M, N, random_ops ? "random" : "zero",
         ms, flops / (ms * 1e-3) / 1e12);
  fflush(stdout);
  sleep(1);
}

int main() {
  long long *d;
  cudaMalloc(&d, 8);
  run<128, 64>(1, d);
  run<128, 64>(0, d);
  run<64, 64>(1, d);
  run<128, 128>(1, d);
  run<64, 128>(1, d);
  run<128, 256>(1, d);
  return 0;
}
