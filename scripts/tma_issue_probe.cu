// Dev probe: is the TMA issue limit per issuing THREAD or per issuing WARP?  Random 16 KB pages
// of a 4 GiB paged pool ([pages, 1 head, 64 tok, 128 d] bf16, SW128 5-D map as the attention
// kernel uses), loaded into SMEM rings that a consumer warp releases immediately.
//   P producer warps x L issuing lanes per warp, each (warp, lane) with its own ring of S stages.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_issue tma_issue_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2605_06914_b200/csrc/taper_internal.cuh"

using namespace taper;

template <int S, int P, int L>
__global__ void __launch_bounds__(64 * P, 1) probe(const __grid_constant__ CUtensorMap tm, const int *order,
                                                   int n_pages, unsigned long long *sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[P * L][S], empty[P * L][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pw = warp % P, role = warp / P;
  if (threadIdx.x == 0) {
    for (int q = 0; q < P * L; ++q)
      for (int i = 0; i < S; ++i) { mbar_init(&full[q][i], 1); mbar_init(&empty[q][i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  if (lane < L) {
    const int q = pw * L + lane;  // ring id
    uint8_t *ring = smem + q * S * 16384;
    unsigned long long acc = 0;
    int n = 0;
    for (long long c = (long long)blockIdx.x * P * L + q; c < n_pages; c += (long long)gridDim.x * P * L, ++n) {
      const int st = n % S;
      if (role == 0) {
        mbar_wait(&empty[q][st], ((n / S) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[q][st], 16384);
        tma_load_5d(ring + st * 16384, &tm, &full[q][st], 0, 0, 0, 0, order[c] % n_pages);
      } else {
        mbar_wait(&full[q][st], (n / S) & 1);
        acc += ring[st * 16384 + (n & 127)];
        mbar_arrive(&empty[q][st]);
      }
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

// each (warp) ring: one 16 KB tile per stage, split into 2 d-halves (8 KB boxes) issued by
// lanes 0 and 1 in the same instruction
template <int S, int P>
__global__ void __launch_bounds__(64 * P, 1) probe_half(const __grid_constant__ CUtensorMap tm, const int *order,
                                                        int n_pages, unsigned long long *sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[P][S], empty[P][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pw = warp % P, role = warp / P;
  if (threadIdx.x == 0) {
    for (int q = 0; q < P; ++q)
      for (int i = 0; i < S; ++i) { mbar_init(&full[q][i], 1); mbar_init(&empty[q][i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  uint8_t *ring = smem + pw * S * 16384;
  unsigned long long acc = 0;
  int n = 0;
  for (long long c = (long long)blockIdx.x * P + pw; c < n_pages; c += (long long)gridDim.x * P, ++n) {
    const int st = n % S;
    if (role == 0) {
      mbar_wait(&empty[pw][st], ((n / S) & 1) ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[pw][st], 16384);
      __syncwarp();
      if (lane < 2) tma_load_5d(ring + st * 16384 + lane * 8192, &tm, &full[pw][st], 0, 0, lane, 0, order[c] % n_pages);
      __syncwarp();
    } else if (lane == 0) {
      mbar_wait(&full[pw][st], (n / S) & 1);
      acc += ring[st * 16384 + (n & 127)];
      mbar_arrive(&empty[pw][st]);
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// the attention kernel's producer structure: one ring per producer warp, warp-uniform loop.
// PAIR = 0: each tile issued by lane (n & 1) (one TMA per instruction);
// PAIR = 1: two consecutive tiles per iteration, issued by lanes 0 and 1 in one instruction
template <int S, int P, int PAIR>
__global__ void __launch_bounds__(64 * P, 1) probe_alt(const __grid_constant__ CUtensorMap tm, const int *order,
                                                       int n_pages, unsigned long long *sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[P][S], empty[P][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pw = warp % P, role = warp / P;
  if (threadIdx.x == 0) {
    for (int q = 0; q < P; ++q)
      for (int i = 0; i < S; ++i) { mbar_init(&full[q][i], 1); mbar_init(&empty[q][i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  uint8_t *ring = smem + pw * S * 16384;
  const long long step = (long long)gridDim.x * P;
  const long long c0 = (long long)blockIdx.x * P + pw;
  if (role == 0) {
    int n = 0;
    for (long long c = c0; c < n_pages; c += (PAIR ? 2 : 1) * step, n += PAIR ? 2 : 1) {
      if (PAIR) {
        const bool two = c + step < n_pages;
        const int my = n + lane;
        const int st = my % S;
        if (lane < (two ? 2 : 1)) {
          mbar_wait(&empty[pw][st], ((my / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[pw][st], 16384);
          tma_load_5d(ring + st * 16384, &tm, &full[pw][st], 0, 0, 0, 0, order[c + lane * step] % n_pages);
        }
        __syncwarp();
      } else {
        const int st = n % S;
        mbar_wait(&empty[pw][st], ((n / S) & 1) ^ 1);
        if (lane == (n & 1)) {
          mbar_arrive_expect_tx(&full[pw][st], 16384);
          tma_load_5d(ring + st * 16384, &tm, &full[pw][st], 0, 0, 0, 0, order[c] % n_pages);
        }
        __syncwarp();
      }
    }
  } else if (lane == 0) {
    unsigned long long acc = 0;
    int n = 0;
    for (long long c = c0; c < n_pages; c += step, ++n) {
      const int st = n % S;
      mbar_wait(&full[pw][st], (n / S) & 1);
      acc += ring[st * 16384 + (n & 127)];
      mbar_arrive(&empty[pw][st]);
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S, int P, int L>
void run(void *pool, const int *order, int n_pages, unsigned long long *sink, int sms) {
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  CUtensorMap tm;
  cuuint64_t dims[5] = {64, 64, 2, 1, (cuuint64_t)n_pages};
  cuuint64_t strides[4] = {256, 128, 256 * 64, 256 * 64};
  cuuint32_t box[5] = {64, 64, 2, 1, 1}, es[5] = {1, 1, 1, 1, 1};
  reinterpret_cast<EncodeFn>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, pool, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto k = probe<S, P, L>;
  const int smem = P * L * S * 16384 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    k<<<sms, 64 * P, smem>>>(tm, order, n_pages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  printf("%d producer warps x %d issuing lanes, %2d stages each (%3d KB in flight/SM): %7.1f GB/s %s\n", P, L, S,
         P * L * S * 16, (double)n_pages * 16384 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

template <int S, int P>
void run_half(void *pool, const int *order, int n_pages, unsigned long long *sink, int sms) {
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  CUtensorMap tm;
  cuuint64_t dims[5] = {64, 64, 2, 1, (cuuint64_t)n_pages};
  cuuint64_t strides[4] = {256, 128, 256 * 64, 256 * 64};
  cuuint32_t box[5] = {64, 64, 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
  reinterpret_cast<EncodeFn>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, pool, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto k = probe_half<S, P>;
  const int smem = P * S * 16384 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    k<<<sms, 64 * P, smem>>>(tm, order, n_pages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  printf("%d producer warps, tile as 2 x 8 KB d-halves from lanes 0/1, %d stages (%3d KB in flight/SM): %7.1f GB/s %s\n",
         P, S, P * S * 16, (double)n_pages * 16384 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

template <int S, int P, int PAIR>
void run_alt(void *pool, const int *order, int n_pages, unsigned long long *sink, int sms) {
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  CUtensorMap tm;
  cuuint64_t dims[5] = {64, 64, 2, 1, (cuuint64_t)n_pages};
  cuuint64_t strides[4] = {256, 128, 256 * 64, 256 * 64};
  cuuint32_t box[5] = {64, 64, 2, 1, 1}, es[5] = {1, 1, 1, 1, 1};
  reinterpret_cast<EncodeFn>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, pool, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto k = probe_alt<S, P, PAIR>;
  const int smem = P * S * 16384 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    k<<<sms, 64 * P, smem>>>(tm, order, n_pages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  printf("%d producer warps, %s, %d stages (%3d KB in flight/SM): %7.1f GB/s %s\n", P,
         PAIR ? "tile pairs from lanes 0/1 in one instruction" : "lane n&1 issues tile n", S, P * S * 16,
         (double)n_pages * 16384 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t pool_bytes = size_t(4) << 30;
  const int n_pages = int(pool_bytes / 16384);
  void *pool;
  int *order;
  unsigned long long *sink;
  cudaMalloc(&pool, pool_bytes);
  cudaMemset(pool, 1, pool_bytes);
  cudaMalloc(&sink, 8);
  std::vector<int> h(n_pages);
  for (int i = 0; i < n_pages; ++i) h[i] = i;
  std::mt19937 rng(1);
  std::shuffle(h.begin(), h.end(), rng);
  cudaMalloc(&order, n_pages * sizeof(int));
  cudaMemcpy(order, h.data(), n_pages * sizeof(int), cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<8, 1, 1>(pool, order, n_pages, sink, sms);
  run<4, 1, 2>(pool, order, n_pages, sink, sms);
  run<2, 1, 4>(pool, order, n_pages, sink, sms);
  run<4, 2, 1>(pool, order, n_pages, sink, sms);
  run<2, 2, 2>(pool, order, n_pages, sink, sms);
  run<5, 2, 1>(pool, order, n_pages, sink, sms);
  run<3, 2, 2>(pool, order, n_pages, sink, sms);
  run<2, 4, 1>(pool, order, n_pages, sink, sms);
  run<3, 4, 1>(pool, order, n_pages, sink, sms);
  run<1, 2, 4>(pool, order, n_pages, sink, sms);
  run<12, 1, 1>(pool, order, n_pages, sink, sms);
  run_half<8, 1>(pool, order, n_pages, sink, sms);
  run_half<4, 2>(pool, order, n_pages, sink, sms);
  run_half<5, 2>(pool, order, n_pages, sink, sms);
  run_alt<4, 2, 0>(pool, order, n_pages, sink, sms);
  run_alt<4, 2, 1>(pool, order, n_pages, sink, sms);
  run_alt<8, 1, 1>(pool, order, n_pages, sink, sms);
  return 0;
}
