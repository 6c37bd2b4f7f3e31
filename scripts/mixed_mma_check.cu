// Dev check: does tcgen05.mma kind::f16 accept A = bf16 and B = fp16 in one instruction
// (instruction descriptor a_format = BF16, b_format = F16)?  One CTA computes
// D[128 x 16] = A[128 x 64] * B[16 x 64]^T with both operands K-major SW128 in SMEM and
// compares with a host fp64 product of the same bf16 / fp16 values.  Also runs the
// same-type bf16 x bf16 case as a control.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mixed_mma mixed_mma_check.cu
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"

using namespace taper;

constexpr int M = 128, N = 16, K = 64;

// generic-store a K-major SW128 operand: row r (128 B = 64 elements), 8-row atoms of 1 KB
__device__ void store_sw128(uint8_t *base, const uint16_t *src, int rows) {
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) {
    const int r = i / 8, c = i % 8;
    const uint4 v = *reinterpret_cast<const uint4 *>(src + r * 64 + c * 8);
    *reinterpret_cast<uint4 *>(base + (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) << 4)) = v;
  }
}

__global__ void __launch_bounds__(128, 1) kern(const uint16_t *a, const uint16_t *b, float *d, int b_f16) {
  __shared__ __align__(1024) uint8_t sA[M * 128];
  __shared__ __align__(1024) uint8_t sB[N * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  store_sw128(sA, a, M);
  store_sw128(sB, b, N);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<32>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    uint32_t idesc = umma_idesc_bf16(M, N, false, false);
    if (b_f16) idesc &= ~(7u << 10);  // b_format = F16 (0)
    const uint64_t a0 = umma_desc_sw128(smem_u32(sA), 16, 1024);
    const uint64_t b0 = umma_desc_sw128(smem_u32(sB), 16, 1024);
    if (lane == 0) {
      for (int kk = 0; kk < 4; ++kk)
        tc_mma_f16(tmem, a0 + uint64_t((kk * 32) >> 4), b0 + uint64_t((kk * 32) >> 4), idesc, kk > 0);
      tc_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[16];
  tmem_ld16(tmem + (uint32_t(warp * 32) << 16), v);
  tmem_ld_wait();
  for (int j = 0; j < N; ++j) d[(warp * 32 + lane) * N + j] = __uint_as_float(v[j]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tmem);
}

int main() {
  std::vector<uint16_t> ha(M * K), hb_bf(N * K), hb_h(N * K);
  std::vector<double> fa(M * K), fb_bf(N * K), fb_h(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) {
    __nv_bfloat16 x = __float2bfloat16(float(rand()) / RAND_MAX * 2.f - 1.f);
    ha[i] = *reinterpret_cast<uint16_t *>(&x);
    fa[i] = __bfloat162float(x);
  }
  for (int i = 0; i < N * K; ++i) {
    const float p = float(rand()) / RAND_MAX;  // softmax-like weights in [0, 1]
    __nv_bfloat16 xb = __float2bfloat16(p);
    __half xh = __float2half(p);
    hb_bf[i] = *reinterpret_cast<uint16_t *>(&xb);
    hb_h[i] = *reinterpret_cast<uint16_t *>(&xh);
    fb_bf[i] = __bfloat162float(xb);
    fb_h[i] = __half2float(xh);
  }
  uint16_t *da, *db;
  float *dd;
  cudaMalloc(&da, M * K * 2);
  cudaMalloc(&db, N * K * 2);
  cudaMalloc(&dd, M * N * 4);
  cudaMemcpy(da, ha.data(), M * K * 2, cudaMemcpyHostToDevice);
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode) {
    const std::vector<uint16_t> &hb = mode ? hb_h : hb_bf;
    const std::vector<double> &fb = mode ? fb_h : fb_bf;
    cudaMemcpy(db, hb.data(), N * K * 2, cudaMemcpyHostToDevice);
    kern<<<1, 128>>>(da, db, dd, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e)); return 2; }
    std::vector<float> hd(M * N);
    cudaMemcpy(hd.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
    double max_err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += fa[m * K + k] * fb[n * K + k];
        max_err = fmax(max_err, fabs(ref - hd[m * N + n]));
      }
    printf("%s: max abs err vs fp64 = %.3e -> %s\n", mode ? "A bf16 x B fp16" : "A bf16 x B bf16 (control)",
           max_err, max_err < 1e-3 ? "OK" : "WRONG");
    fails += max_err >= 1e-3;
  }
  return fails ? 1 : 0;
}
