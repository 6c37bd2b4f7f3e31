// Dev check of the operand layouts the row-mode attention path uses (one CTA, 128 threads):
//   QK:  S[M x 64]   = Q[M x 128] K[64 x 128]^T   A = Q (SMEM, K-major SW128, 8-row groups 2 KB
//        apart, d-halves 1 KB apart), B = K tile (SMEM, K-major SW128, [d-half][64][128 B])
//   PV:  O[M x 128] += P[M x 64] V[64 x 128]      A = P (TMEM, bf16 pairs, written with
//        tcgen05.st), B = V tile (SMEM, MN-major SW128, [d-half][64 tokens][128 B])
// for M = 128 (row r in TMEM lane r) and M = 64 (row r in lane 32 (r / 16) + r % 16, read and
// written with the 16x32bx2 shape: thread t < 16 lane t columns [c, c + n), t >= 16 lane t - 16
// columns [c + IMM, ...)).  Compares with host fp64 products.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o rowmode rowmode_check.cu
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"

using namespace taper;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// q [128 rows][128 d], k [64][128], v [64][128], p [128][64] (bf16 bits)
template <int M>
__global__ void __launch_bounds__(128, 1) kern(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                               const uint16_t *p, float *s_out, float *o_out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sQ = sm;                 // 32 KB: [branch 16][d-half][8 rows][128 B]
  uint8_t *sK = sm + 32768;         // 16 KB: [d-half][64 tokens][128 B]
  uint8_t *sV = sm + 49152;         // 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 16; i += 128) {  // Q: row r, 16-B chunk c (8 per d-half)
    const int r = i / 16, c = i % 16, hf = c / 8, cc = c % 8;
    const uint4 val = *reinterpret_cast<const uint4 *>(q + r * 128 + c * 8);
    *reinterpret_cast<uint4 *>(sQ + (r / 8) * 2048 + hf * 1024 + (r % 8) * 128 + ((cc ^ (r % 8)) << 4)) = val;
  }
  for (int i = tid; i < 64 * 16; i += 128) {  // K / V: token t, chunk c
    const int t = i / 16, c = i % 16, hf = c / 8, cc = c % 8;
    const int off = hf * 8192 + (t / 8) * 1024 + (t % 8) * 128 + ((cc ^ (t % 8)) << 4);
    *reinterpret_cast<uint4 *>(sK + off) = *reinterpret_cast<const uint4 *>(k + t * 128 + c * 8);
    *reinterpret_cast<uint4 *>(sV + off) = *reinterpret_cast<const uint4 *>(v + t * 128 + c * 8);
  }
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lane_off = uint32_t(warp * 32) << 16;
  const uint32_t tS = tmem, tP = tmem + 384, tO = tmem + 128;
  // P -> TMEM (row-major P[row][64 tokens] as 32 columns of bf16 pairs)
  {
    uint32_t pk[32];
    if (M == 128) {
      const int row = warp * 32 + lane;
      for (int j = 0; j < 32; ++j) pk[j] = uint32_t(p[row * 64 + 2 * j]) | (uint32_t(p[row * 64 + 2 * j + 1]) << 16);
      tmem_st_n<32>(tP + lane_off, pk);
    } else {
      const int row = warp * 16 + (lane & 15), half = lane >> 4;
      for (int j = 0; j < 16; ++j) {
        const int tk = 32 * half + 2 * j;
        pk[j] = uint32_t(p[row * 64 + tk]) | (uint32_t(p[row * 64 + tk + 1]) << 16);
      }
      tmem_st_x2_8<16>(tP + lane_off, pk);
      tmem_st_x2_8<16>(tP + lane_off + 8, pk + 8);  // columns [8, 16) and [24, 32)
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint32_t idesc_qk = umma_idesc_bf16(M, 64, false, false);
    const uint32_t idesc_pv = umma_idesc_bf16(M, 128, false, true);
    const uint64_t a0 = umma_desc_sw128(smem_u32(sQ), 16, 2048);
    const uint64_t b0 = umma_desc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t v0 = umma_desc_sw128(smem_u32(sV), 8192, 1024);
    if (lane == 0) {
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t a = a0 + uint64_t((((kk >> 2) * 1024) + (kk & 3) * 32) >> 4);
        const uint64_t b = b0 + uint64_t((((kk >> 2) * 8192) + (kk & 3) * 32) >> 4);
        tc_mma_f16(tS, a, b, idesc_qk, kk > 0);
      }
      for (int kk = 0; kk < 4; ++kk)
        mma_ts(tO, tP + kk * 8, v0 + uint64_t((kk * 2048) >> 4), idesc_pv, kk > 0);
      tc_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (M == 128) {
    const int row = warp * 32 + lane;
    uint32_t v32[32];
    for (int c = 0; c < 2; ++c) {
      tmem_ld32(tS + lane_off + 32 * c, v32);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) s_out[row * 64 + 32 * c + j] = __uint_as_float(v32[j]);
    }
    for (int c = 0; c < 4; ++c) {
      tmem_ld32(tO + lane_off + 32 * c, v32);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) o_out[row * 128 + 32 * c + j] = __uint_as_float(v32[j]);
    }
  } else {
    const int row = warp * 16 + (lane & 15), half = lane >> 4;
    uint32_t v32[32];
    tmem_ld_x2_32<32>(tS + lane_off, v32);  // t<16: cols [0,32); t>=16: [32,64)
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) s_out[row * 64 + 32 * half + j] = __uint_as_float(v32[j]);
    for (int c = 0; c < 2; ++c) {
      tmem_ld_x2_32<64>(tO + lane_off + 32 * c, v32);  // t<16: [32c, +32); t>=16: [64+32c, +32)
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) o_out[row * 128 + 64 * half + 32 * c + j] = __uint_as_float(v32[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

static uint16_t bf(float x, double *back) {
  __nv_bfloat16 h = __float2bfloat16(x);
  *back = __bfloat162float(h);
  return *reinterpret_cast<uint16_t *>(&h);
}

template <int M>
int run() {
  std::vector<uint16_t> q(128 * 128), k(64 * 128), v(64 * 128), p(128 * 64);
  std::vector<double> fq(q.size()), fk(k.size()), fv(v.size()), fp(p.size());
  srand(7 + M);
  auto rnd = [] { return float(rand()) / RAND_MAX * 2.f - 1.f; };
  for (size_t i = 0; i < q.size(); ++i) q[i] = bf(rnd(), &fq[i]);
  for (size_t i = 0; i < k.size(); ++i) k[i] = bf(rnd(), &fk[i]);
  for (size_t i = 0; i < v.size(); ++i) v[i] = bf(rnd(), &fv[i]);
  for (size_t i = 0; i < p.size(); ++i) p[i] = bf(float(rand()) / RAND_MAX, &fp[i]);
  uint16_t *dq, *dk, *dv, *dp;
  float *ds, *dO;
  cudaMalloc(&dq, q.size() * 2); cudaMalloc(&dk, k.size() * 2); cudaMalloc(&dv, v.size() * 2);
  cudaMalloc(&dp, p.size() * 2); cudaMalloc(&ds, 128 * 64 * 4); cudaMalloc(&dO, 128 * 128 * 4);
  cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, k.data(), k.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v.data(), v.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, p.data(), p.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  kern<M><<<1, 128, 66 * 1024>>>(dq, dk, dv, dp, ds, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("M=%d: CUDA error %s\n", M, cudaGetErrorString(e)); return 1; }
  std::vector<float> s(128 * 64), o(128 * 128);
  cudaMemcpy(s.data(), ds, s.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0;
  for (int r = 0; r < M; ++r) {
    for (int t = 0; t < 64; ++t) {
      double ref = 0;
      for (int d = 0; d < 128; ++d) ref += fq[r * 128 + d] * fk[t * 128 + d];
      es = fmax(es, fabs(ref - s[r * 64 + t]));
    }
    for (int d = 0; d < 128; ++d) {
      double ref = 0;
      for (int t = 0; t < 64; ++t) ref += fp[r * 64 + t] * fv[t * 128 + d];
      eo = fmax(eo, fabs(ref - o[r * 128 + d]));
    }
  }
  printf("M=%d: QK max abs err %.3e (%s), PV(TS) max abs err %.3e (%s)\n", M, es, es < 1e-3 ? "OK" : "WRONG",
         eo, eo < 1e-3 ? "OK" : "WRONG");
  return (es < 1e-3 && eo < 1e-3) ? 0 : 1;
}

int main() { return run<128>() | run<64>(); }
