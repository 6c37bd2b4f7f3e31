// Dev microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M=128) cost per instruction
// for the shapes the attention kernel uses.  One CTA; warp 0 issues (elect.sync, warp-
// uniform operands, fully unrolled), commits to an mbarrier and waits; clock64 deltas.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"

using namespace taper;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

template <int N, bool TS, int CHAINS, bool MASK, int COUNT>
__global__ void __launch_bounds__(128, 1) bench(long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (48 * 1024) / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t sA = smem_u32(smem);
    const uint32_t sB = smem_u32(smem + 16384);
    constexpr uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    uint32_t mask[4] = {0u, 0u, 0u, 0u};
    if (MASK) { mask[1] = mask[2] = mask[3] = 0xffffffffu; }
    const uint64_t a0 = umma_desc_sw128(sA, 16, 1024), b0 = umma_desc_sw128(sB, 16, 1024);
    if (elect_one()) {
      for (int i = 0; i < 8; ++i) tc_mma_f16(tmem, a0, b0, idesc, 0u);
      tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    long long t0 = clock64();
    if (elect_one()) {
#pragma unroll
      for (int i = 0; i < COUNT; ++i) {
        const uint32_t d = tmem + (i % CHAINS) * N;
        const uint64_t b = b0 + uint64_t(((i & 3) * 32) >> 4);
        if (TS) {
          tc_mma_f16_ts(d, tmem + 256 + (i & 7) * 8, b, idesc, 1u, mask);
        } else {
          const uint64_t a = a0 + uint64_t(((i & 3) * 32) >> 4);
          tc_mma_f16(d, a, b, idesc, 1u);
        }
      }
      tc_commit(&bar);
    }
    __syncwarp();
    long long t1 = clock64();
    mbar_wait(&bar, 1);
    long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, bool TS, int CHAINS, bool MASK>
void run(long long *d_out) {
  constexpr int COUNT = 64;
  auto k = bench<N, TS, CHAINS, MASK, COUNT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  long long h[2];
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 128, 50 * 1024>>>(d_out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  }
  cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
  printf("%4d %3d %6d %4d %18.1f %18.1f %6d\n", N, int(TS), CHAINS, int(MASK),
         double(h[0]) / COUNT, double(h[1]) / COUNT, 128 * N / 256);
}

int main() {
  long long *d_out;
  cudaMalloc(&d_out, 16);
  printf("   N  TS chains mask  cycles/MMA(issue)  cycles/MMA(total)  floor\n");
  run<64, false, 1, false>(d_out);
  run<64, false, 2, false>(d_out);
  run<64, false, 4, false>(d_out);
  run<128, false, 1, false>(d_out);
  run<128, false, 2, false>(d_out);
  run<256, false, 1, false>(d_out);
  run<64, true, 1, false>(d_out);
  run<64, true, 2, false>(d_out);
  run<128, true, 1, false>(d_out);
  run<128, true, 2, false>(d_out);
  run<128, true, 1, true>(d_out);
  run<256, true, 1, false>(d_out);
  run<32, false, 1, false>(d_out);
  run<16, false, 1, false>(d_out);
  run<16, false, 8, false>(d_out);
  return 0;
}
